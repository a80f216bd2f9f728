"""Summarise an ncu --set full report into profiles/: per-kernel key metrics + top stall reasons,
and the DRAM traffic per launch that bench.py reports as roofline.traffic.

usage: python tools/ncu_summary.py gpurun_out/<tag>_full.ncu-rep profiles/<tag>_ncu_full_summary.json
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "lts__t_sector_hit_rate.pct",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, out = sys.argv[1], Path(sys.argv[2])
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    stall = [i for i, h in enumerate(hdr)
             if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    summary, traffic = {}, {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mpmgpu::", "")
        ent = {k: float(d[k]) for k in KEYS if d.get(k) not in (None, "")}
        ent["units"] = {k: units[hdr.index(k)] for k in KEYS if k in hdr}
        st = sorted(((float(r[i] or 0), hdr[i][len("smsp__average_warps_issue_stalled_"):-len(
            "_per_issue_active.ratio")]) for i in stall), reverse=True)[:6]
        ent["top_stalls_per_issue"] = {n: round(v, 3) for v, n in st}
        summary.setdefault(name, []).append(ent)
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[k]) * SCALE.get(units[hdr.index(k)], 1.0)
        short = next((k for k in ("k_p2g", "k_g2p", "k_grid", "k_inc_block", "k_inc_scan", "k_inc_classify")
                      if name.startswith(k)), name)
        traffic[short] = {"dram_bytes": b, "kernel": name, "source": Path(rep).name}
        if d.get("lts__t_sector_hit_rate.pct") not in (None, ""):
            traffic[short]["l2_hit_rate_pct"] = float(d["lts__t_sector_hit_rate.pct"])
    out.write_text(json.dumps(summary, indent=1))
    tp = out.parent / "traffic.json"
    old = json.loads(tp.read_text()) if tp.exists() else {}
    old.update(traffic)
    tp.write_text(json.dumps(old, indent=1))
    print(json.dumps({k: v["dram_bytes"] for k, v in traffic.items()}))


if __name__ == "__main__":
    main()
