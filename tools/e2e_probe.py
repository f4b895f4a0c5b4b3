"""End-to-end (host buffers) variance probe at 128^3: the pipelined host API
(Assembler.assemble_async, 3 fields in flight) timed over K steps, R repeats,
with the process pinned or not to the GPU's NUMA-local cores (NVML).
Output: one JSON line.  Used for bench.py's e2e setup."""
import json
import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def local_cpus():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = [64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
        return cpus
    except Exception as e:  # pragma: no cover
        return None


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "any"
    out = {"mode": mode, "nproc": os.cpu_count()}
    cpus = local_cpus()
    out["gpu_local_cpus"] = f"{len(cpus)} cpus {cpus[:4]}..{cpus[-2:]}" if cpus else None
    if mode == "local" and cpus:
        os.sched_setaffinity(0, cpus)
    import paper_2403_08777_b200 as tb
    from paper_2403_08777_b200 import _native as N
    mesh = tb.generate_box_mesh(128, 128, 128)
    u = tb.make_velocity(mesh, "random:1")
    asm = tb.Assembler(mesh, tb.RunConfig(scatter="private-atomic"))
    P = tb.PhysParams()
    n = mesh.coords.shape[0]
    pu = [N.PinnedArray((n, 3)) for _ in range(4)]
    pr = [N.PinnedArray((n, 3)) for _ in range(4)]
    for p in pu:
        p.array[:] = u
    for i in range(8):
        asm.wait(asm.assemble_async(pu[i % 4].array, P, pr[i % 4].array, "private-atomic"))
    res = []
    for k in (50, 200, 200, 200, 50):
        t = time.perf_counter()
        tk = [asm.assemble_async(pu[i % 4].array, P, pr[i % 4].array, "private-atomic") for i in range(k)]
        for x in tk[-4:]:
            asm.wait(x)
        res.append((k, round(mesh.connectivity.shape[0] * k / (time.perf_counter() - t) / 1e9, 3)))
    out["gelem_s"] = res
    try:
        out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-600:]
    except Exception:
        pass
    print(json.dumps(out))


main()
