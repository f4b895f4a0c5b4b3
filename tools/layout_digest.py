"""SHA-256 digests of the host layout (tal_plan_blobs: chunk blobs, blob
offsets, node permutation) over a set of meshes x layout options.  Written
once by the serial preprocessing (round 1 code) into
tests/golden/layout_digests.json; tests/test_layout.py checks that the
multithreaded preprocessing reproduces every layout bit for bit.

    python tools/layout_digest.py [--write]
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2403_08777_b200 as tb  # noqa: E402
from paper_2403_08777_b200.mesh import plan_blobs  # noqa: E402

import os  # noqa: E402

# TAL_RING_SORT=0 (patches in build order inside each chunk) is the layout the
# round-1 serial code wrote; the default sorts each chunk's patches by ring
# length and has its own record
OUT = ROOT / "tests" / "golden" / ("layout_digests.json" if os.environ.get("TAL_RING_SORT") == "0"
                                   else "layout_digests_ringsort.json")


def cases():
    box = tb.generate_box_mesh(24, 20, 18)
    perm = tb.permute_nodes(tb.generate_box_mesh(14, 13, 12),
                            np.random.default_rng(0).permutation(15 * 14 * 13))
    for name, m in (("box24x20x18", box), ("perm14x13x12", perm)):
        for ren in ("rcm", "sfc", "none"):
            for eo in ("sfc", "node", "keep"):
                yield f"{name}/{ren}/{eo}", m, tb.RunConfig(renumber=ren, element_order=eo)
        for cp, cn in ((64, 144), (256, 512), (100, 200), (7, 16)):
            yield f"{name}/cta{cp}/cn{cn}", m, tb.RunConfig(cta_patches=cp, chunk_nodes=cn)
        yield f"{name}/tet", m, tb.RunConfig(patches="tet")
    yield "box64/default", tb.generate_box_mesh(64, 64, 64), tb.RunConfig()


def digest(m, cfg) -> str:
    d = plan_blobs(m, cfg)
    h = hashlib.sha256()
    for k in ("blobs", "blob_off", "perm"):
        a = d[k]
        h.update(b"-" if a is None else np.ascontiguousarray(a).tobytes())
    h.update(str(d["threads"]).encode())
    return h.hexdigest()


def compute() -> dict:
    return {k: digest(m, cfg) for k, m, cfg in cases()}


if __name__ == "__main__":
    got = compute()
    if "--write" in sys.argv:
        OUT.write_text(json.dumps(got, indent=1) + "\n")
        print("wrote", OUT, len(got))
    else:
        want = json.loads(OUT.read_text())
        bad = [k for k in want if want[k] != got.get(k)]
        print("mismatch:", bad if bad else "none", f"({len(want)} cases)")
