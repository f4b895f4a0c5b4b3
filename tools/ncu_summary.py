"""Summarise an ncu --set full report: headline metrics + stall breakdown.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "?")
    g = lambda k: d.get(k, "")
    def f(k):
        try:
            return float(g(k).replace(",", ""))
        except ValueError:
            return None
    def mb(k):  # byte-valued metric in MB whatever unit ncu chose
        v = f(k)
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}
        return None if v is None else v * scale.get(units[hdr.index(k)], 1.0)

    def tot(op):
        r = f(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum")
        if r is not None:
            return r
        r = f(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
        c = f("smsp__cycles_elapsed.avg")
        return None if r is None or c is None else round(r * c)

    stalls = {}
    for k in hdr:
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", k)
        if m and f(k):
            stalls[m.group(1)] = round(f(k), 3)
    s = {
        "kernel": name,
        "duration": [f("gpu__time_duration.sum"), units[hdr.index("gpu__time_duration.sum")]],
        "sm_clock": [f("smsp__cycles_elapsed.avg.per_second"),
                     units[hdr.index("smsp__cycles_elapsed.avg.per_second")]],
        "dram_read_mbytes": mb("dram__bytes_read.sum"),
        "dram_write_mbytes": mb("dram__bytes_write.sum"),
        "fp64_pipe_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "warps_active_per_sm": f("sm__warps_active.avg.per_cycle_active"),
        "registers": f("launch__registers_per_thread"),
        "smem_per_block": f("launch__shared_mem_per_block_dynamic"),
        "inst_executed": f("smsp__inst_executed.sum"),
        # the full set reports these as rates: x elapsed SM cycles = totals
        "dfma_thread_inst": tot("dfma"),
        "dmul_thread_inst": tot("dmul"),
        "dadd_thread_inst": tot("dadd"),
        "local_ld_inst": f("sass__inst_executed_local_loads"),
        "local_st_inst": f("sass__inst_executed_local_stores"),
        "lsu_pipe_pct": f("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        "shared_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "shared_bank_conflicts": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
        "l2_sectors": f("lts__t_sectors.sum"),
        "l2_throughput_pct": f("lts__t_sectors.avg.pct_of_peak_sustained_elapsed"),
        "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "l1_hit_pct": f("l1tex__t_sector_hit_rate.pct"),
        "red_sectors": f("l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum"),
        "stalls_per_issue": dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10]),
    }
    out[name] = s
for name, s in out.items():
    print(json.dumps(s, indent=1))
if "--json" in sys.argv:
    json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
