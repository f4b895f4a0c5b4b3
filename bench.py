#!/usr/bin/env python
"""bench.py -- assembled elements/s of the P1-tet momentum-RHS assembly on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (BASELINE.json config 2): a 128^3 Kuhn box (12,582,912 tets,
2,146,689 nodes), random:1 velocity (uniform [-1,1), default_rng(1)),
PhysParams defaults, RCM node renumbering + Morton element order.  Under
torchrun (N>1) every rank assembles its own 128^3 slab of a 128x128x(128N)
box and the interface planes are summed over NCCL (weak scaling).

One step = one full RHS assembly (zero/merge + element kernel) with inputs
resident in HBM, replayed as one captured CUDA graph at N=1 (``--no-graph``:
direct launches); L2 is flushed (256 MiB write) before every step, outside
the CUDA-event-timed interval.  ``e2e`` repeats the step through the public
host API (pinned host u -> H2D -> assembly -> D2H rhs) and times it by wall
clock.  ``--impl reference`` times the reference algorithm's CPU port
(oracle/, the threaded private driver of variants.py:573-596) on all host
cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FLOP_PER_ELEM = 448  # reference RSP ledger, variants.py:207-217 (cli.py:182 convention)
NOMINAL_FP64_TFLOPS = 37.2  # 148 SM x 64 DFMA/clk x 2 x 1.965 GHz


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cells", type=int, default=None,
                    help="cells per side: of each rank's slab (--scaling weak; default 128, "
                         "config 2 at N=1; 160 = config 5) or of the whole box split over the "
                         "ranks (--scaling strong; default 256 = config 4)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="N>1: weak = a cells^3 slab per rank of a cells x cells x (cells N) box; "
                         "strong = one cells^3 box cut into N z-slabs")
    ap.add_argument("--init", default="random:1")
    ap.add_argument("--scatter", default="private-atomic")
    ap.add_argument("--variant", choices=["rsp", "rs", "b", "p"], default="rsp",
                    help="code shape (rs/b: the paper's study shapes, one thread per element)")
    ap.add_argument("--renumber", default="rcm")
    ap.add_argument("--element-order", default="sfc")
    ap.add_argument("--patches", default="star")
    ap.add_argument("--cta-patches", type=int, default=128)
    ap.add_argument("--chunk-nodes", type=int, default=256)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="N=1: launch each step's zeroing + kernel directly instead of replaying "
                         "one captured CUDA graph per step (tal_graph_capture)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--permute", action="store_true", help="config 3: random node permutation")
    ap.add_argument("--mesh", default="box",
                    help="box (Kuhn box of --cells) | delaunay:NPOINTS (unstructured: the Delaunay "
                         "tetrahedralisation of NPOINTS seeded random points; N=1 only)")
    ap.add_argument("--pressure", action="store_true",
                    help="add the P1 pressure-gradient term (extension; uniform [-1,1) nodal p, seed 2)")
    ap.add_argument("--supg", action="store_true",
                    help="add the SUPG stabilisation term (extension; c1=4, c2=2)")
    ap.add_argument("--partition", choices=["slab", "rcb"], default="slab",
                    help="N>1: z-slabs of the box (weak scaling) or RCB of the (optionally "
                         "--permute'd) global box mesh, exchange-path interface sum")
    ap.add_argument("--check", action="store_true",
                    help="N>1: gather the owned RHS rows to rank 0 and check them against the oracle")
    return ap.parse_args()


def cells_of(a) -> int:
    return a.cells if a.cells is not None else (256 if a.scaling == "strong" else 128)


def self_launch(a) -> int | None:
    """``--gpus N`` without a torchrun environment: re-launch this command as
    N ranks under torch.distributed.run (127.0.0.1 rendezvous, a free port)
    and return its exit code; None when this process is already a rank.  A
    torchrun world that disagrees with --gpus is refused."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != a.gpus:
            sys.exit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={ws}; refusing a mismatched run")
        return None
    if a.gpus <= 1:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, ValueError):
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, smax, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if s > 500] or sm
        return {
            "sm_mhz": statistics.median(load) if load else None,
            "sm_max_mhz": max(smax) if smax else None,
            "power_w_max": max(pw) if pw else None,
            "samples": len(sm),
            "reasons": sorted(reasons),
        }


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU path on all host cores
# ---------------------------------------------------------------------------
def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def import_reference():
    """tet-assembly-lab from baseline/_ref (pip-installed copy, git-ignored,
    travels to the GPU box; numba is part of the image), else None."""
    base = ROOT / "baseline" / "_ref"
    if not (base / "tet_assembly_lab").is_dir():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tal_numba_cache")
    if str(base) not in sys.path:
        sys.path.append(str(base))
    try:
        import tet_assembly_lab as ref
        from tet_assembly_lab import harness, variants
        return ref, variants, harness
    except Exception:  # numba or numpy missing / incompatible
        return None


def reference_cpu(cells, init: str, steps: int, warmup: int, budget_s: float = 120.0) -> dict:
    """Time the reference's own RSP assembly on the host: its harness
    ``run_bench(mesh, u, VariantId.RSP, PhysParams(), RunConfig(n_threads=T,
    scatter='private', reps=steps), verify=False)`` (harness.py:75-128, the
    survey's CPU-baseline recipe), T = all host threads; the
    value is the harness's own median-based elem/s.  The sample is the
    (nx, ny, nz) box ``cells``, cut to fewer z layers when the whole run would
    exceed ``budget_s``.  Falls back to the C port of the numba kernel
    (oracle/, bitwise equal to it) when the reference cannot be imported."""
    T = host_threads()
    nx, ny, nz = cells
    R = import_reference()
    if R is not None:
        ref, variants, harness = R
        P = ref.PhysParams()
        cfg1 = variants.RunConfig(n_threads=T, scatter="private", reps=1)
        probe = ref.generate_box_mesh(nx, ny, max(1, min(nz, 8)))
        up = ref.make_velocity(probe, init)
        variants.assemble_rsp(probe, up, P, cfg1)  # numba JIT / cache load
        t = variants.assemble_rsp(probe, up, P, cfg1).wall_time / probe.n_elems
        per_step = t * 6 * nx * ny * nz
        total = max(steps, 1) + max(warmup, 0) + 1
        if per_step * total > budget_s:
            nz = max(1, int(nz * budget_s / (per_step * total)))
        mesh = ref.generate_box_mesh(nx, ny, nz)
        u = ref.make_velocity(mesh, init)
        for _ in range(max(warmup, 0)):
            variants.assemble_rsp(mesh, u, P, cfg1)
        rec, _ = harness.run_bench(mesh, u, variants.VariantId.RSP, P,
                                   variants.RunConfig(n_threads=T, scatter="private",
                                                      reps=max(steps, 1)), verify=False)
        return {"value": rec.melems_per_s * 1e6, "unit": "elem/s", "cores": T, "kind": "reference",
                "steps": rec.reps, "median_s": rec.median_time,
                "sample": f"{nx}x{ny}x{nz} Kuhn box ({mesh.n_elems} tets), {init}; the reference "
                          f"package (tet-assembly-lab 0.1.0, numba) harness.run_bench, RSP, "
                          f"scatter=private, n_threads={T}, 1 warm-up + {max(warmup, 0)} + median of "
                          f"{rec.reps}"}
    from oracle import oracle as O
    O.build()
    m = O.box_mesh(nx, ny, nz)
    u = O.velocity(m.coords, init)
    O.assemble_rsp(m.coords, m.connectivity, u, n_threads=T)
    t0 = time.perf_counter()
    O.assemble_rsp(m.coords, m.connectivity, u, n_threads=T)
    per_step = time.perf_counter() - t0
    total = max(steps, 1) + max(warmup, 0)
    E = m.n_elems
    sample_elems = E if per_step * total <= budget_s else max(int(E * budget_s / (per_step * total)), 6)
    conn = np.ascontiguousarray(m.connectivity[:sample_elems])
    for _ in range(max(warmup, 0)):
        O.assemble_rsp(m.coords, conn, u, n_threads=T)
    ts = []
    for _ in range(max(steps, 1)):
        t0 = time.perf_counter()
        O.assemble_rsp(m.coords, conn, u, n_threads=T)
        ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    return {"value": sample_elems / med, "unit": "elem/s", "cores": T, "kind": "port",
            "steps": len(ts), "median_s": med,
            "sample": f"{'all' if sample_elems == E else 'first %d of the' % sample_elems} "
                      f"{E} tets of a {nx}x{ny}x{nz} Kuhn box, {init}; C port of "
                      f"_rsp_kernels.assemble_elements + the variants.py private driver "
                      f"(reference not importable), {T} threads, median of {len(ts)}"}


def run_reference(a) -> None:
    """``--impl reference``: rank 0 alone times the reference's own CPU path on
    the host cores on the sample of one rank's share of our arm's workload
    (N=1: the whole config-2 box); the other ranks exit without work."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    c = cells_of(a)
    gz = c * ws if a.scaling == "weak" else c
    local_z = gz // ws if ws > 1 else gz
    cb = reference_cpu((c, c, max(local_z, 1)), a.init, a.steps, a.warmup)
    if ws == 1:
        workload = f"{c}^3 Kuhn box, {a.init}"
    elif a.scaling == "weak":
        workload = f"{c}x{c}x{gz} Kuhn box, a {c}^3 slab per rank ({ws} ranks), {a.init}"
    else:
        cut = "z-slabs" if a.partition == "slab" else "RCB parts"
        workload = f"{c}^3 Kuhn box cut into {ws} {cut}" + (" (random node numbering)" if a.permute else "") + \
            f", {a.init}"
    line = {
        "impl": "reference", "metric": "assembled elements/s", "value": cb["value"],
        "unit": "elem/s", "n_gpus": ws, "steps": cb["steps"], "warmup": a.warmup,
        "ms_per_step": 1e3 * cb["median_s"], "higher_is_better": True, "scaling": a.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "box_cells": [c, c, gz], "host_only": True},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "elem/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def measured_hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6532.9, "MEASURED_PEAKS.json value at round start (file absent on this box)"


def traffic_key(a, workload: str) -> str:
    """profiles/traffic.json key: the workload AND everything that changes the
    kernel's memory behaviour (node numbering, element order, chunking)."""
    return (f"{workload} | permuted={int(bool(a.permute))} renumber={a.renumber} "
            f"element_order={a.element_order} patches={a.patches} cta={a.cta_patches} "
            f"chunk_nodes={a.chunk_nodes} pressure={int(bool(a.pressure))} supg={int(bool(a.supg))}")


def ncu_traffic(kernel_key: str, key: str) -> dict:
    """ncu --set full figures for this exact configuration (tools/update_traffic.py),
    or {} when none was captured."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        return dict(json.loads(p.read_text()).get(key, {}).get(kernel_key) or {})
    except Exception:
        return {}


def run_ours(a) -> None:
    import torch

    import paper_2403_08777_b200 as tb
    from paper_2403_08777_b200 import _native as N

    ws, rank, local = dist_env()
    dev = local % max(torch.cuda.device_count(), 1)  # ranks may share a GPU in validation runs
    torch.cuda.set_device(dev)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        # gloo: host-staged validation runs with ranks time-sharing fewer GPUs
        # (NCCL refuses two ranks on one device)
        backend = os.environ.get("TAL_DIST_BACKEND",
                                 "nccl" if torch.cuda.device_count() >= ws else "gloo")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    P = tb.PhysParams()
    cfg = tb.RunConfig(scatter=a.scatter, renumber=a.renumber, element_order=a.element_order,
                       patches=a.patches, cta_patches=a.cta_patches, chunk_nodes=a.chunk_nodes,
                       device=dev)
    c = cells_of(a)
    gz = c * ws if a.scaling == "weak" else c  # global box: (c, c, gz)
    if gz < ws:
        raise SystemExit(f"bench.py: {gz} cell layers cannot be split over {ws} ranks")
    if a.mesh != "box" and ws > 1:
        raise SystemExit("bench.py: --mesh delaunay runs on one GPU (N=1)")
    t0 = time.perf_counter()
    gperm = None
    if ws > 1 and a.partition == "rcb":
        from paper_2403_08777_b200.distributed import PartitionedDomain
        g = tb.generate_box_mesh(c, c, gz)
        if a.permute:
            gperm = np.random.default_rng(0).permutation(g.n_nodes)
            g = tb.permute_nodes(g, gperm)
        dom = PartitionedDomain(g, rank, ws, cfg)
        mesh, u = dom.mesh, dom.set_velocity(tb.make_velocity(g, a.init))
        asm = dom.assembler
        del g
    elif ws > 1:
        from paper_2403_08777_b200.distributed import SlabDomain
        dom = SlabDomain((c, c, gz), rank, ws, cfg)
        mesh, u = dom.mesh, dom.velocity(a.init)
        asm = dom.assembler
    elif a.mesh.startswith("delaunay"):
        dom = None
        mesh = tb.generate_delaunay_mesh(int(a.mesh.partition(":")[2] or 2_000_000), seed=0)
        u = tb.make_velocity(mesh, a.init)
        asm = tb.Assembler(mesh, cfg, build_colors=(a.scatter == "colored"))
    else:
        dom = None
        mesh = tb.generate_box_mesh(c, c, c)
        if a.permute:
            mesh = tb.permute_nodes(mesh, np.random.default_rng(0).permutation(mesh.n_nodes))
        u = tb.make_velocity(mesh, a.init)
        asm = tb.Assembler(mesh, cfg, build_colors=(a.scatter == "colored" or (
            a.variant != "rsp" and a.scatter == "private")))
    prep_s = time.perf_counter() - t0
    info = asm.info()
    press = None
    if a.pressure:
        press = np.random.default_rng(2).uniform(-1.0, 1.0, mesh.n_nodes)
        asm.set_pressure(press)
    if a.supg:
        asm.set_stabilization(True)
    E, Nn = mesh.n_elems, mesh.n_nodes

    stream = torch.cuda.current_stream().cuda_stream

    use_graph = not a.no_graph and dom is None

    def one_step():
        if use_graph:
            return asm.replay(stream=stream)
        if dom is None:
            return asm.run(P, stream=stream, variant=a.variant)
        return dom.step(P, stream=stream)

    parity = None
    cpu_baseline = None

    asm.set_velocity_host(u, stream=stream)
    flush_buf = None if a.no_flush else torch.empty(64 * 1024 * 1024, dtype=torch.int32,
                                                    device=f"cuda:{dev}")

    def flush():
        if flush_buf is not None:
            flush_buf.fill_(1)

    if use_graph:
        asm.capture(P, variant=a.variant)
    asm.profile(True)
    for _ in range(max(a.warmup, 0)):
        flush()
        one_step()
    torch.cuda.synchronize()
    asm.profile_read()
    fp64_tf, fp64_mhz = N.fp64_peak(dev, 5.0)  # >= 5 ms DFMA launches, best of 20
    gpus_shared = torch.cuda.device_count() < ws
    if gpus_shared:  # ranks time-sharing one GPU probe concurrently: each sees a fraction
        fp64_tf = NOMINAL_FP64_TFLOPS

    sampler = ClockSampler(dev)
    sampler.start()
    time.sleep(0.15)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    launches = 0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for i in range(a.steps):
        flush()
        starts[i].record()
        launches += one_step()
        ends[i].record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    wall1 = time.perf_counter()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kern_ms = asm.profile_read()
    fused = dom is not None and dom.fused
    if use_graph or fused or not len(kern_ms):
        # a replayed graph carries no profile events: time the dominant kernel
        # in plain launches of the same step (with peers attached a plain run
        # is the whole fused step: every rank runs the same count)
        for _ in range(min(a.steps, 50)):
            flush()
            if dom is None or fused:
                asm.run(P, stream=stream, variant=a.variant)
            else:
                dom.step(P, stream=stream)
        torch.cuda.synchronize()
        kern_ms = asm.profile_read()
    # nvidia-smi polls the driver every 50 ms: stop it before the wall-clock
    # e2e leg (observed to depress e2e to 9-10 Gelem/s from 11.6)
    clocks = sampler.stop()
    total_ms = float(sum(step_ms))
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    E_all = E * ws
    kmean = float(np.mean(kern_ms))
    step_mean = float(np.mean(step_ms))
    rate = E / (kmean * 1e-3)  # dominant-kernel elements/s of this GPU
    bytes_per_elem = (16 * E + 72 * Nn) / E if E else 0.0
    if dist:  # whole-job elements; slowest rank's kernel, step and kernel rate
        e = torch.tensor([float(E)], device=f"cuda:{dev}", dtype=torch.float64)
        t = torch.tensor([kmean, step_mean], device=f"cuda:{dev}", dtype=torch.float64)
        r = torch.tensor([rate], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(r, op=dist.ReduceOp.MIN)
        E_all, kmean, step_mean, rate = int(e.item()), float(t[0].item()), float(t[1].item()), \
            float(r.item())
    units = E_all * a.steps
    value = units / (total_ms * 1e-3)

    # device-resident in the CALLER's layout: a solver that keeps u and rhs as
    # (N,3) AoS device arrays in its own node numbering pays the layout
    # conversion every step: set_velocity_device (k_pack_velocity, renumbered
    # gather) -> assembly -> get_rhs_device (k_unpack_aos); CUDA events
    caller_layout = None
    if dom is None and a.variant == "rsp":
        u_dev = torch.as_tensor(u, device=f"cuda:{dev}").contiguous()
        r_dev = torch.empty_like(u_dev)
        ks = max(min(a.steps, 100), 3)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * ks)]
        def timed(step):
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            for i in range(ks):
                flush()
                ev[2 * i].record()
                step()
                ev[2 * i + 1].record()
            torch.cuda.synchronize()
            return float(np.mean([ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(ks)]))

        def composed():
            asm.set_velocity_device(u_dev.data_ptr(), stream=stream)
            one_step()
            asm.get_rhs_device(r_dev.data_ptr(), stream=stream)

        def fused():
            asm.run_caller(P, u_dev.data_ptr(), r_dev.data_ptr(), scatter=a.scatter, stream=stream)

        cl_ms = timed(fused)
        comp_ms = timed(composed)
        caller_layout = {"value": E / (cl_ms * 1e-3), "unit": "elem/s", "ms_per_step": cl_ms,
                         "steps": ks,
                         "api": "Assembler.run_caller (tal_run_caller): the private kernel gathers u from "
                                "and writes rhs to the caller's (N,3) device arrays in its own node "
                                "numbering; CUDA events, L2 flushed between steps",
                         "composed_ms_per_step": comp_ms,
                         "composed_api": "set_velocity_device (pack) -> step -> get_rhs_device (unpack)"}
        del u_dev, r_dev
    # end-to-end through the public host API (pinned host buffers): every step
    # copies that step's u host->device and reads its rhs back device->host.
    #  sync     : Assembler.assemble_into (one field at a time, blocking)
    #  pipelined: Assembler.assemble_async, three fields in flight (H2D of the
    #             next field and D2H of the previous result overlap the assembly)
    e2e = None
    if not a.no_e2e and dom is None and a.variant == "rsp":
        NSLOT = 4  # >= tal_handle::ASYNC_SLOTS: a host buffer is never reused while in flight
        pu = [N.PinnedArray((Nn, 3)) for _ in range(NSLOT)]
        pr = [N.PinnedArray((Nn, 3)) for _ in range(NSLOT)]
        for p_ in pu:
            p_.array[:] = u
        ksteps = max(min(a.steps, 200), 3)
        for _ in range(2):
            asm.assemble_into(pu[0].array, P, pr[0].array, a.scatter)
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(ksteps):
            flush()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            asm.assemble_into(pu[0].array, P, pr[0].array, a.scatter)
            tot += time.perf_counter() - t1
        sync_val = E * ksteps / tot
        for i in range(2 * NSLOT):  # warm the async slots
            asm.wait(asm.assemble_async(pu[i % NSLOT].array, P, pr[i % NSLOT].array, a.scatter))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        tickets = [asm.assemble_async(pu[i % NSLOT].array, P, pr[i % NSLOT].array, a.scatter)
                   for i in range(ksteps)]
        for tk in tickets[-NSLOT:]:
            asm.wait(tk)
        pipe_tot = time.perf_counter() - t1
        ok = bool(np.array_equal(pr[0].array, pr[1].array)) if a.scatter in ("private", "colored") \
            else bool(np.allclose(pr[0].array, pr[1].array, rtol=0, atol=1e-12 * np.abs(pr[0].array).max()))
        e2e = {"value": E * ksteps / pipe_tot, "unit": "elem/s", "h2d_bytes_per_step": 24 * Nn,
               "d2h_bytes_per_step": 24 * Nn, "steps": ksteps,
               "api": "Assembler.assemble_async (tal_assemble_async): 3 fields in flight, "
                      "H2D/D2H overlapped with the assembly; wall clock over all steps",
               "sync_value": sync_val,
               "sync_api": "Assembler.assemble_into (tal_assemble), one field at a time, wall clock",
               "pipelined_results_consistent": ok}
        for p_ in pu + pr:
            p_.free()
    if not a.no_e2e and dom is not None:
        # N>1: every rank copies its slab's u host->device (pinned), runs the
        # step (assembly + interface sum), reads its rhs back; max over ranks.
        # Fused interface sum: the step is one tal_run, so the pipelined host
        # API (tal_assemble_async, 3 fields in flight) carries it; exchange
        # path: one blocking round trip per step (the NCCL exchange sits
        # between the assembly and the D2H).
        NSLOT = 4
        pu = [N.PinnedArray((Nn, 3)) for _ in range(NSLOT)]
        pr = [N.PinnedArray((Nn, 3)) for _ in range(NSLOT)]
        for p_ in pu:
            p_.array[:] = u
        ksteps = max(min(a.steps, 50), 3)
        if dom.fused:
            for i in range(2 * NSLOT):
                asm.wait(asm.assemble_async(pu[i % NSLOT].array, P, pr[i % NSLOT].array, a.scatter))
        else:
            for _ in range(2):
                asm.set_velocity_host(pu[0].array, stream=stream)
                one_step()
                asm.get_rhs_host(pr[0].array, stream=stream)
        torch.cuda.synchronize()
        dist.barrier()
        t1 = time.perf_counter()
        if dom.fused:
            tickets = [asm.assemble_async(pu[i % NSLOT].array, P, pr[i % NSLOT].array, a.scatter)
                       for i in range(ksteps)]
            for tk in tickets[-NSLOT:]:
                asm.wait(tk)
        else:
            for _ in range(ksteps):
                asm.set_velocity_host(pu[0].array, stream=stream)
                one_step()
                asm.get_rhs_host(pr[0].array, stream=stream)
                torch.cuda.synchronize()
        tt = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": E * ws * ksteps / float(tt.item()), "unit": "elem/s",
               "h2d_bytes_per_step": 24 * Nn * ws, "d2h_bytes_per_step": 24 * Nn * ws,
               "steps": ksteps,
               "api": ("Assembler.assemble_async on each rank's slab (fused interface sum inside "
                       "the step), 3 fields in flight" if dom.fused else
                       "SlabDomain.step with Assembler.set_velocity_host / get_rhs_host per rank")
                      + " (pinned), wall clock, max over ranks"}
        for p_ in pu + pr:
            p_.free()
    # the numba seam swapped inside the reference's OWN driver:
    # tet_assembly_lab.variants.assemble_rsp with _rsp_kernels.assemble_elements
    # -> paper_2403_08777_b200.assemble_elements (tal_seam_*), timed by the
    # reference's own wall_time (variants.py:572, :616); one-thread driver (one
    # call with ids = all elements) and the threaded private driver (one call
    # per vector_dim-aligned slab, numpy merge of the per-thread buffers)
    seam = None
    R = import_reference() if (dom is None and a.variant == "rsp" and not a.no_e2e
                               and a.scatter in ("private", "private-atomic")) else None
    if R is not None:
        ref, variants, _ = R
        from tet_assembly_lab import _rsp_kernels
        orig = _rsp_kernels.assemble_elements
        seam_s = [0.0]

        def timed_seam(*args):
            t1 = time.perf_counter()
            tb.assemble_elements(*args)
            seam_s[0] += time.perf_counter() - t1

        _rsp_kernels.assemble_elements = timed_seam
        try:
            seam = {"unit": "elem/s", "api": "reference variants.assemble_rsp (scatter='private') with "
                    "_rsp_kernels.assemble_elements swapped for paper_2403_08777_b200.assemble_elements; "
                    "the reference's own wall_time, median of 5 after 2 warm-ups",
                    "h2d_bytes_per_step": 24 * Nn, "d2h_bytes_per_step": 24 * Nn}
            for T in (1, host_threads()):
                cfgr = variants.RunConfig(n_threads=T, scatter="private")
                for _ in range(2):
                    variants.assemble_rsp(mesh, u, ref.PhysParams(), cfgr)
                seam_s[0] = 0.0
                ws_ = [variants.assemble_rsp(mesh, u, ref.PhysParams(), cfgr).wall_time for _ in range(5)]
                seam[f"threads_{T}"] = {"value": E / statistics.median(ws_),
                                        "ms_per_step": 1e3 * statistics.median(ws_),
                                        "seam_calls_ms_per_step": 1e3 * seam_s[0] / 5}
            seam["value"] = seam["threads_1"]["value"]
        finally:
            _rsp_kernels.assemble_elements = orig
            tb.clear_cache()
    # parity + CPU baseline (rank 0, N=1): the oracle as checker / baseline only.
    # Runs after the e2e leg, so its 16-thread host load cannot disturb it.
    if ws == 1 and not a.no_cpu_baseline:
        from oracle import oracle as O
        O.build()
        rhs_gpu, _ = asm.assemble(u, P, variant=a.variant)
        # bounded sample of the same workload on all host cores (the reference's
        # own numba path when importable); the oracle's vector is the checker
        cpu_baseline = None if a.mesh != "box" else reference_cpu((c, c, c), a.init, 3, 0, budget_s=30.0)
        ref = O.assemble_rsp(mesh.coords, mesh.connectivity, u, n_threads=O.default_threads())
        if press is not None:
            ref = ref + O.pressure_gradient(mesh.coords, mesh.connectivity, press)
        if a.supg:
            ref = ref + O.supg_term(mesh.coords, mesh.connectivity, u)
        chk = O.compare(rhs_gpu, ref, mesh.coords, mesh.connectivity, u)
        parity = {"reference_rel_diff": chk.rel_diff, "rel_l2": chk.rel_l2,
                  "entry_rel": chk.entry_rel, "passed": bool(chk.passed)}
    if dom is not None and a.check:  # N>1 parity: owned rows of every rank vs the oracle
        torch.cuda.synchronize()
        rows = [None] * ws
        dist.all_gather_object(rows, dom.owned_rhs())
        if rank == 0:
            from oracle import oracle as O
            O.build()
            g = O.box_mesh(c, c, gz)
            if gperm is not None:  # the permuted global mesh the ranks partitioned
                gm = tb.permute_nodes(tb.Mesh(coords=g.coords, connectivity=g.connectivity), gperm)
                g = O.OracleMesh(np.ascontiguousarray(gm.coords), np.ascontiguousarray(gm.connectivity))
            ug = O.velocity(g.coords, a.init)
            ref = O.assemble_rsp(g.coords, g.connectivity, ug, n_threads=O.default_threads())
            full = np.full_like(ref, np.nan)
            for ids, blk in rows:
                full[ids] = blk
            chk = O.compare(full, ref, g.coords, g.connectivity, ug)
            parity = {"reference_rel_diff": chk.rel_diff, "rel_l2": chk.rel_l2,
                      "entry_rel": chk.entry_rel, "passed": bool(chk.passed),
                      "gathered": f"owned rows of {ws} ranks vs single-domain oracle"}
    asm.profile(False)

    if a.mesh.startswith("delaunay"):
        workload = (f"unstructured: Delaunay of {mesh.n_nodes} random points in the unit cube "
                    f"({mesh.n_elems} tets), {a.init}")
    elif ws == 1:
        workload = f"{c}^3 Kuhn box, {a.init}"
    elif a.scaling == "weak":
        workload = f"{c}x{c}x{gz} Kuhn box, a {c}^3 slab per rank ({ws} ranks), {a.init}"
    else:
        cut = "z-slabs" if a.partition == "slab" else "RCB parts"
        workload = f"{c}^3 Kuhn box cut into {ws} {cut}" + (" (random node numbering)" if a.permute else "") + \
            f", {a.init}"
    tf = FLOP_PER_ELEM * rate / 1e12  # per GPU (the slowest rank at N>1)
    alg_bytes = 16 * E + 72 * Nn  # int32 conn + coords/u read + rhs write
    hbm_gbs = bytes_per_elem * rate / 1e9
    hbm_peak, hbm_src = measured_hbm_peak()
    kname = {"private": "k_assemble_private<cfg,ordered=true>",
             "private-atomic": "k_assemble_private<cfg,ordered=false>",
             "atomic": "k_assemble_atomic<true>", "colored": "k_assemble_colored<true> (all colours)",
             "sequential": "k_assemble_sequential (reference order, strict IEEE)"}[a.scatter]
    if a.variant != "rsp":
        colored = a.scatter in ("private", "colored")
        kname = {"b": "k_assemble_baseline", "p": "k_assemble_baseline<fixed>",
                 "rs": "k_assemble_rs"}[a.variant] + \
            ("<colored> (all colours)" if colored else "<atomic>")
    tr = ncu_traffic(kname, traffic_key(a, workload))
    traffic = tr.get("dram_bytes_per_launch")
    line = {
        "metric": "assembled elements/s", "value": value, "unit": "elem/s", "n_gpus": ws,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": total_ms / a.steps,
        "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated Kuhn box mesh, seeded velocity)",
        "config": {"workload": workload, "n_elems": E_all, "n_elems_rank0": E, "n_nodes_rank0": Nn,
                   "box_cells": [c, c, gz] if a.mesh == "box" else None, "mesh": a.mesh,
                   "scatter": a.scatter,
                   "renumber": a.renumber, "element_order": a.element_order,
                   "patches": a.patches, "cta_patches": a.cta_patches, "chunk_nodes": a.chunk_nodes,
                   "permuted": bool(a.permute), "variant": a.variant,
                   "pressure_term": bool(a.pressure), "supg_term": bool(a.supg),
                   "cuda_graph": bool(use_graph),
                   "l2": "flushed (256 MiB write) before every step, outside the timed events"
                         if flush_buf is not None else "not flushed",
                   "gpus_shared": gpus_shared,
                   "traffic_key": traffic_key(a, workload),
                   "parallelism": (f"dp{ws} z-slabs" if a.partition == "slab" else f"dp{ws} RCB parts")
                   if ws > 1 else "single GPU",
                   "interface_sum": None if dom is None else (
                       "fused: assembly kernel REDs into the neighbours' RHS (CUDA IPC peer memory)"
                       if dom.fused else "exchange: NCCL send/recv of the interface planes + halo add"
                       + (f" (fused unavailable: {dom.fused_error})" if dom.fused_error else ""))},
        "roofline": {"bound": "fp64", "kernel": kname, "achieved": tf, "peak": fp64_tf,
                     "unit": "TFLOP/s", "frac": tf / fp64_tf,
                     "peak_source": ("nominal 148 SM x 64 DFMA/clk x 2 x 1965 MHz: the ranks share one "
                                     "GPU, so a live probe would see a fraction of the pipe (validation "
                                     "line, not a performance claim)") if gpus_shared else (
                                    "live DFMA probe in this run (tal_fp64_peak: >= 5 ms "
                                    "launches of 8 independent DFMA chains per thread, best of 20, at "
                                    f"{fp64_mhz:.0f} MHz measured in-kernel); DFMA issues at ~58.3 of "
                                    "the nominal 64 lanes/clk/SM while DMUL/DADD reach 63.8 "
                                    "(tools/probe_fp64.cu, profiles/round2/probe_fp64.txt); nominal "
                                    f"{NOMINAL_FP64_TFLOPS} at 1965 MHz"),
                     "frac_of_nominal": tf / NOMINAL_FP64_TFLOPS,
                     "probe_sm_mhz": fp64_mhz,
                     "flop_per_elem": FLOP_PER_ELEM, "kernel_ms": kmean,
                     "per": "GPU" if ws == 1 else "GPU (slowest rank's kernel rate)",
                     "step_ms_mean": step_mean,
                     "non_kernel_ms_per_step": step_mean - kmean,
                     "traffic": traffic,
                     "traffic_source": tr.get("source"),
                     "l2_sector_bytes": tr.get("l2_sector_bytes_per_launch"),
                     "hbm": {"achieved": hbm_gbs, "peak": hbm_peak,
                             "unit": "GB/s", "frac": hbm_gbs / hbm_peak,
                             "alg_bytes_per_launch": alg_bytes, "peak_source": hbm_src}},
        "e2e": e2e,
        "device_caller_layout": caller_layout,
        "seam_in_reference_driver": seam,
        "cpu_baseline": cpu_baseline,
        "parity": parity,
        "gpu_launches": launches,
        "clocks": clocks,
        "prep": {"seconds": prep_s, "native_prep_seconds": info["prep_seconds"],
                 "n_patches": info["n_patches"], "n_chunks": info["n_chunks"],
                 "n_chunk_nodes": info["n_chunk_nodes"],
                 "n_shared_nodes": info["n_shared_nodes"], "device_bytes": info["device_bytes"]},
        "wall_s_timed_region": wall1 - wall0,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    asm.close() if dom is None else dom.close()
    if dist:
        dist.destroy_process_group()


def main():
    a = parse()
    rc = self_launch(a)
    if rc is not None:
        sys.exit(rc)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
