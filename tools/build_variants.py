"""Build A/B variants of libtal_b200.so into build/var/<name>.so.

    python tools/build_variants.py name=DEF1,DEF2 name2=DEF3 ...   ("base" = no defines)

Each variant is timed on the GPU by tools/gpu_variants.sh (bench.py with
TAL_LIB_PATH pointing at it)."""
import shutil
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2403_08777_b200 import build as B  # noqa: E402

out = ROOT / "build" / "var"
if "--keep" not in sys.argv:
    shutil.rmtree(out, ignore_errors=True)
out.mkdir(parents=True, exist_ok=True)
specs = []
for a in [x for x in sys.argv[1:] if x != "--keep"]:
    name, _, defs = a.partition("=")
    specs.append((name, [d for d in defs.split(",") if d]))


def one(spec):
    name, defs = spec
    B.build(out=out / f"{name}.so", defines=defs, tag=f"_{name}")
    return name


with ThreadPoolExecutor(4) as ex:
    for n in ex.map(one, specs):
        print("built", n)
