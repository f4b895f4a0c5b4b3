"""B200 code-shape study table (PAPER.md:254-291
on A100) from the ncu summaries and bench lines in profiles/round1/shapes/.

    python tools/shape_study.py [dir]   -> dir/study.json + markdown table on stdout
"""
import json
import sys
from pathlib import Path

D = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/round1/shapes")
E = 12582912  # 128^3 Kuhn box
rows = [("B", "ncu_b.json", "bench_shape_b_atomic.json"),
        ("P (study only)", "ncu_p.json", "bench_shape_p_atomic.json"),
        ("RS", "ncu_rs.json", "bench_shape_rs_atomic.json"),
        ("RSP thread/tet", "ncu_rsp_atomic.json", "bench_shape_rsp_atomic.json"),
        ("RSP edge-star (production)", "../ncu_full_private_atomic.json", "../bench_default.json")]
out = []
for label, prof, bench in rows:
    s = next(iter(json.loads((D / prof).read_text()).values()))
    b = json.loads((D / bench).read_text().strip().splitlines()[-1])
    flop = (2 * s["dfma_thread_inst"] + s["dmul_thread_inst"] + s["dadd_thread_inst"]) / E
    dram = (s["dram_read_mbytes"] + s["dram_write_mbytes"]) * 1e6 / E
    kms = b["roofline"]["kernel_ms"]
    out.append({"shape": label, "kernel_ms": kms, "gelem_s": E / kms / 1e6,
                "ncu_ms": s["duration"][0] * (1.0 if s["duration"][1] == "ms" else 1e-3),
                "registers": s["registers"], "local_ld_st": [s["local_ld_inst"], s["local_st_inst"]],
                "exec_flop_per_elem": flop, "dram_bytes_per_elem": dram,
                "exec_gflops": flop * E / kms / 1e6, "fp64_pipe_pct": s["fp64_pipe_pct"],
                "issue_active_pct": s["issue_active_pct"]})
(D / "study.json").write_text(json.dumps(out, indent=1))
print("| shape | kernel ms | Gelem/s | regs | FP64 flop/elem (executed) | DRAM B/elem | GFlop/s (executed) | FP64 pipe |")
print("|---|---|---|---|---|---|---|---|")
for r in out:
    print(f"| {r['shape']} | {r['kernel_ms']:.3f} | {r['gelem_s']:.2f} | {r['registers']:.0f} | "
          f"{r['exec_flop_per_elem']:.0f} | {r['dram_bytes_per_elem']:.1f} | {r['exec_gflops']:.0f} | "
          f"{r['fp64_pipe_pct']:.1f}% |")
