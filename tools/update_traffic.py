"""Regenerate profiles/traffic.json (bench.py's roofline.traffic and
l2_sector_bytes) from pairs of (bench JSON line, ncu --set full summary of
the same command): the bench line names its configuration key
(config.traffic_key) and dominant kernel, the summary holds
dram__bytes_read.sum + dram__bytes_write.sum and lts__t_sectors.sum of one
launch.  Usage: python tools/update_traffic.py bench.json ncu.json [...]"""
import json
import sys
from pathlib import Path

R = Path(__file__).resolve().parent.parent
out_p = R / "profiles" / "traffic.json"
out = json.loads(out_p.read_text()) if out_p.exists() else {}
args = sys.argv[1:]
if len(args) % 2:
    sys.exit(__doc__)
for bj, nj in zip(args[0::2], args[1::2]):
    line = json.loads(Path(bj).read_text().strip().splitlines()[-1])
    key, kern = line["config"]["traffic_key"], line["roofline"]["kernel"]
    summ = json.loads(Path(nj).read_text())
    s = next(v for k, v in summ.items() if "k_assemble" in k)
    ent = {"dram_bytes_per_launch": (s["dram_read_mbytes"] + s["dram_write_mbytes"]) * 1e6,
           "source": f"{Path(nj).resolve().relative_to(R)} (ncu --set full: dram__bytes_read.sum + "
                     "dram__bytes_write.sum; lts__t_sectors.sum x 32 B)"}
    if s.get("l2_sectors") is not None:
        ent["l2_sector_bytes_per_launch"] = s["l2_sectors"] * 32.0
    out.setdefault(key, {})[kern] = ent
    print(key, kern, ent)
out_p.write_text(json.dumps(out, indent=1) + "\n")
