"""Per-kernel SASS instruction counts of the product library (cuobjdump -sass):
tcgen05.mma (UTCHMMA), TMA loads (UTMALDG), TMEM loads (LDTM), tcgen05
commits/barriers (UTCBAR), legacy mma.sync (HMMA), ldmatrix (LDSM), cp.async
(LDGSTS), local-memory spill traffic (STL/LDL) -- the evidence that each hot
kernel runs on the sm_100a tensor-core / TMA path.

Usage: python scripts/sass_summary.py [--lib paper_2505_01572_b200/libpipespec.so] [--out profiles/r02_sass_summary.json]
"""
import argparse
import collections
import json
import re
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default="paper_2505_01572_b200/libpipespec.so")
ap.add_argument("--out", default=None)
a = ap.parse_args()
sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
OPS = ("UTCHMMA", "UTMALDG", "LDTM", "UTCBAR", "HMMA", "LDSM", "LDGSTS", "SYNCS", "STL", "LDL", "ATOM")
cnt = collections.defaultdict(collections.Counter)
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    for op in OPS:
        if re.search(r"\b" + op + r"\b", line):
            cnt[cur][op] += 1
out = {k: dict(v) for k, v in sorted(cnt.items()) if k.startswith("_ZN2ps")}
print(json.dumps(out, indent=1))
if a.out:
    json.dump(out, open(a.out, "w"), indent=1)
