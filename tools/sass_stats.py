"""Per-kernel SASS opcode histogram of libtal_b200.so (cuobjdump -sass).

    python tools/sass_stats.py [regex] [--so path]

Counts static instructions per function, grouped by pipe-relevant classes
(FP64: DFMA/DMUL/DADD/DSETP/MUFU; memory: LDG/LDS/STS/STG/REDG/ATOMS; ...).
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

so = Path(__file__).resolve().parent.parent / "paper_2403_08777_b200" / "libtal_b200.so"
args = [a for a in sys.argv[1:]]
if "--so" in args:
    i = args.index("--so")
    so = Path(args[i + 1])
    del args[i:i + 2]
pat = re.compile(args[0]) if args else None
out = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True, check=True).stdout
funcs = {}
cur = None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[0-9T]\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and cur:
        funcs[cur][m.group(1) + (m.group(2) or "")] += 1
for name, c in funcs.items():
    if pat and not pat.search(name):
        continue
    base = Counter()
    for k, v in c.items():
        base[k.split(".")[0]] += v
    fp64 = sum(base[k] for k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
    print(f"== {name}  total={sum(c.values())}  fp64={fp64}")
    print("   " + "  ".join(f"{k}:{v}" for k, v in base.most_common(24)))
    wide = {k: v for k, v in c.items() if k.split(".")[0] in ("LDG", "STG", "REDG", "LDS", "STS", "ATOMS", "ATOMG")}
    print("   mem: " + "  ".join(f"{k}:{v}" for k, v in sorted(wide.items())))
