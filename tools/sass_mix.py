"""Per-kernel SASS instruction mix of libsplatct.so (cuobjdump -sass): the
tensor-core, TMA and async-copy instructions that show which hardware paths a
kernel uses.

    python tools/sass_mix.py > profiles/sass_mix.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2411_04844_b200", "_lib", "libsplatct.so")
KEYS = ["HMMA", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "LDGSTS",
        "SYNCS", "FFMA2", "FFMA", "DFMA", "LDS", "LDG", "STG", "ATOMS", "ATOMG", "RED", "SHFL"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
rows = []
for blk in funcs[1:]:
    name = blk.split("\n", 1)[0].strip()
    demangled = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    cnt = collections.Counter()
    for line in blk.splitlines():
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            op = m.group(1)
            cnt[op] += 1
    mix = {k: sum(v for op, v in cnt.items() if op == k or op.startswith(k + "."))
           for k in KEYS}
    rows.append((demangled, sum(cnt.values()), mix))
print("# SASS instruction mix per kernel of libsplatct.so (static counts, cuobjdump -sass)")
print("# kernel | total | " + " ".join(KEYS))
for name, tot, mix in sorted(rows):
    short = re.sub(r"\(.*", "", name)
    nz = " ".join(f"{k}={v}" for k, v in mix.items() if v)
    print(f"{short:60s} total={tot:6d} {nz}")
