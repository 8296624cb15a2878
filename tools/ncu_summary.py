"""Summarise ncu reports into profiles/ (run here, on the CPU box):
    python tools/ncu_summary.py <report.ncu-rep> <workload> <out-name>
Writes profiles/<out-name>.txt (key metrics per kernel) and merges DRAM
traffic per launch into profiles/traffic.json (read by bench.py)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__average_warp_latency_per_inst_issued.ratio",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
]
STALLS = "smsp__average_warp_latency_issue_stalled"


def main():
    rep, workload, name = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    traffic = {}
    for r in data:
        d = dict(zip(hdr, r))
        kname = d.get("Kernel Name", "?")
        out.append(f"== {kname}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k} = {d[k]} {units[hdr.index(k)]}")
        st = sorted(((k, d[k]) for k in hdr if k.startswith(STALLS) and k.endswith(".ratio")),
                    key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]
        for k, v in st:
            out.append(f"  stall {k[len(STALLS) + 1:]} = {v}")
        try:
            rb = float(d["dram__bytes_read.sum"].replace(",", "")) * (1024 ** 2 if "M" in units[hdr.index("dram__bytes_read.sum")] else 1)
        except Exception:
            rb = None
        out.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", name + ".txt"), "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
