# GPU: stencil SpMM parity tests + SpMM timings on the C2/C3/C4 shapes (CSR vs stencil twin)
out=${1:-gpurun_out/stencil}
timeout 600 python -m pytest tests/test_gpu_stencil.py -x -q > $out.tests.log 2>&1; echo rc=$? >> $out.tests.log
tail -3 $out.tests.log
for h in "" --hint; do
 timeout 120 python tools/spmm_time.py --kind convdiff7 --grid 128 --m 8 $h
 timeout 200 python tools/spmm_time.py --kind stencil27 --grid 192 --m 16 --seed 2 $h
 timeout 300 python tools/spmm_time.py --kind convdiff7 --grid 320 --m 32 --seed 3 --reps 10 $h
done 2>&1 | tee $out.time.log
