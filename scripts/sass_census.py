"""SASS instruction census of the built library (tcgen05 / TMA / MUFU evidence), per kernel.

usage: python scripts/sass_census.py [libdfb200.so] > profiles/r2_sass_census.json
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2601_20499_b200", "libdfb200.so")
MNEMONICS = ["UTCHMMA", "UTCHMMA.2CTA", "UTCBAR", "UTCBAR.2CTA", "LDTM", "STTM", "UTMALDG", "UTMAPF", "MUFU.EX2",
             "FFMA2", "FADD2", "FMNMX3", "SYNCS.ARRIVE", "SYNCS.PHASECHK"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
out, cur = {}, None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        out[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(1)
    for mn in MNEMONICS:
        if op == mn or op.startswith(mn + "."):
            out[cur][mn] += 1
demangled = {}
for k, v in out.items():
    try:
        name = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    except OSError:
        name = k
    if any(v.values()):
        demangled[name] = dict(sorted(v.items()))
json.dump({"library": os.path.relpath(lib, ROOT), "tool": "cuobjdump -sass",
           "note": "a mnemonic counts its suffixed forms too (UTCHMMA includes UTCHMMA.2CTA)", "kernels": demangled},
          sys.stdout, indent=1)
print()
