"""Summarise `nvcc -Xptxas -v` logs: kernel, registers, stack, spills."""
import re
import subprocess
import sys

for path in sys.argv[1:]:
    text = open(path).read()
    blocks = re.split(r"ptxas info\s+: Compiling entry function '", text)[1:]
    for b in blocks:
        name = b.split("'", 1)[0]
        try:
            dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        except OSError:
            dem = name
        dem = re.sub(r"\(.*", "", dem).replace("hk::", "")
        regs = re.search(r"Used (\d+) registers", b)
        stack = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", b)
        print(f"{dem:45s} regs={regs.group(1) if regs else '?':>4s} "
              f"stack={stack.group(1) if stack else '?':>5s} spill_st={stack.group(2) if stack else '?':>4s} "
              f"spill_ld={stack.group(3) if stack else '?':>4s}")
