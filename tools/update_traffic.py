"""Regenerate profiles/traffic.json (bench.py's roofline.traffic) from the
ncu --set full summaries in profiles/round1/ (dram read + write per launch)."""
import json
from pathlib import Path

R = Path(__file__).resolve().parent.parent / "profiles"
src = {
    "k_assemble_private<cfg,ordered=false>": "round1/ncu_full_private_atomic.json",
    "k_assemble_private<cfg,ordered=true>": "round1/ncu_full_private_ordered.json",
    "k_assemble_atomic<true>": "round1/shapes/ncu_rsp_atomic.json",
    "k_assemble_rs<atomic>": "round1/shapes/ncu_rs.json",
    "k_assemble_baseline<atomic>": "round1/shapes/ncu_b.json",
}
out = {}
for k, f in src.items():
    s = next(iter(json.loads((R / f).read_text()).values()))
    out[k] = {"dram_bytes_per_launch": (s["dram_read_mbytes"] + s["dram_write_mbytes"]) * 1e6,
              "source": f"profiles/{f} (ncu --set full: dram__bytes_read.sum + dram__bytes_write.sum)"}
(R / "traffic.json").write_text(json.dumps({"128^3 Kuhn box, random:1": out}, indent=1) + "\n")
print(json.dumps(out, indent=1))
