"""bench.py host logic (CPU): partitions, the shared config record, the
reference arm's independence from the product library, and the --gpus N
launcher refusing to measure fewer GPUs than asked."""
import json
import os
import subprocess
import sys
from argparse import Namespace
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def _args(**kw):
    base = dict(config="C3", method=None, m=None, tol=None, fixed=None, maxit=None, formulation="fused")
    base.update(kw)
    return Namespace(**base)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_whole_planes(world):
    cfg = bench.resolve(_args())
    b = bench.partition(cfg, world)
    plane = 192 * 192
    assert b[0] == 0 and b[-1] == 192 ** 3 and len(b) == world + 1
    assert all(x % plane == 0 for x in b)
    assert all(b[i + 1] - b[i] >= plane for i in range(world))
    sizes = [(b[i + 1] - b[i]) // plane for i in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_partition_banded_rows():
    cfg = bench.resolve(_args(config="C5"))
    b = bench.partition(cfg, 8)
    assert b == [i * 1_000_000 for i in range(9)]


def test_resolve_overrides():
    cfg = bench.resolve(_args(config="C4"))
    assert cfg["fixed"] and cfg["maxit"] == 200 and cfg["m"] == 32 and cfg["method"] == "pipebicgstab"
    cfg = bench.resolve(_args(config="C5", m=32, fixed=50))
    assert cfg["m"] == 32 and cfg["maxit"] == 50 and cfg["fixed"]
    cfg = bench.resolve(_args(config="C2", method="rbicgstab"))
    assert cfg["method"] == "rbicgstab" and not cfg["fixed"] and cfg["tol"] == 1e-8


def test_config_record_is_shared():
    cfg = bench.resolve(_args())
    c1 = bench.config_dict(cfg, 4, 189_119_224)
    assert c1["rows"] == 192 ** 3 and c1["m"] == 16 and c1["method"] == "rbicgstab"
    assert c1 == bench.config_dict(bench.resolve(_args()), 4, 189_119_224)


def test_reference_arm_never_loads_the_product():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "0", "--cpu-iters", "3"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["product_library_loaded"] is False
    cfg = bench.resolve(_args(config="C1"))
    assert line["config"] == bench.config_dict(cfg, 1, line["config"]["nnz"])
    assert line["config"]["nnz"] == 223_232
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0


def test_gpus_n_refuses_without_devices():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("box has >= 2 GPUs")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert out.returncode == 2
    assert "refusing" in out.stderr
