"""Static SASS opcode histogram of one kernel: python tools/sass_mix.py <obj|so> <mangled-substring>"""
import re
import subprocess
import sys
from collections import Counter

obj, pat = sys.argv[1], sys.argv[2]
text = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", text)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = Counter()
    for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", f):
        ops[m.group(2)] += 1
    total = sum(ops.values())
    dp = sum(v for k, v in ops.items() if k in ("DADD", "DMUL", "DFMA"))
    print(f"{name}: {total} instrs, DP(add/mul/fma)={dp}, MUFU={ops['MUFU']}, STG={ops['STG']}, CALL={ops['CALL']}")
    print("   ", ", ".join(f"{k}:{v}" for k, v in ops.most_common(25)))
