"""Print registers / spills per kernel from the build's ptxas -v logs."""
import glob
import re
import subprocess
import sys

for log in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "build/obj/*.ptxas.log")):
    fn = None
    spill = ""
    for line in open(log):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            fn = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            spill = f"spill {m.group(1)}/{m.group(2)}"
        m = re.search(r"Used (\d+) registers", line)
        if m and fn:
            print(f"{m.group(1):>4} regs  {spill:16s} {fn[:110]}")
            fn = None
