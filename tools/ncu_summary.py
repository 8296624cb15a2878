"""Summarise ncu reports into profiles/ (run in the build container):

    python tools/ncu_summary.py <report.ncu-rep> <workload> <out-name> [--per-launch-units N]

Writes profiles/<out-name>.txt (key metrics + top stall reasons per kernel)
and merges DRAM traffic per launch (dram__bytes_read.sum +
dram__bytes_write.sum) into profiles/traffic.json, which bench.py reports
as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
]
STALL = "smsp__average_warp_latency_issue_stalled_"
NAME_MAP = {"k_rs_contract_expand": "rs5_expand", "k_rs_contract_link": "rs3_link", "k_rs_select": "rs2_select",
            "k_cc_part_scatter2": "cc_partition_scatter","k_rs_walk_stage": "rs3_walk", "k_rs_walk_bin": "rs3_walk",
            "k_rs_top_jump": "rs4_rank", "k_rs_top_init": "rs4_rank", "k_rs_top_coop": "rs4_rank", "k_spl_meta_block": "splitter_meta", "k_rs_walk_rec": "rs3_walk", "k_rs_walk<sg::Level0": "rs3_walk",
            "k_rs_walk<Level0": "rs3_walk", "k_rs_walk<sg::LevelK": "rs4_walk", "k_rs_walk<LevelK": "rs4_walk",
            "k_rs_rec_refine": "rs5_refine", "k_rs_refine_atom": "rs5_refine", "k_rs_refine_lean": "rs5_refine",
            "k_cc_part_chunks": "cc_partition", "k_rs_rec_scatter": "rs5_scatter", "k_rs_rec_partition": "rs5_partition",
            "k_rs_expand0": "rs5_expand", "k_rs_count0": "rs1_validate", "k_cc_hook_uf": "cc_hook_uf",
            "k_cc_hook_sv": "cc_hook_sv", "k_cc_part_scatter": "cc_partition_scatter",
            "k_cc_part_count": "cc_partition_count", "k_wy_jump": "wy_jump", "k_cc_compress": "cc_shortcut"}


def value(d, units, hdr, k):
    try:
        v = float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None
    return v * SCALE.get(units[hdr.index(k)], 1)


def short(kname):
    if "k_rs_contract<" in kname:  # <SuccT, kVec>
        return "rs3_contract"
    for pat, nm in NAME_MAP.items():
        if pat in kname:
            return nm
    return kname.split("(")[0].split("<")[0].replace("void ", "")


def main():
    rep, workload, name = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = [f"# ncu --set full summary: {os.path.basename(rep)} ({workload})", ""]
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    seen = set()
    for r in data:
        d = dict(zip(hdr, r))
        kname = d.get("Kernel Name", "?")
        out.append(f"== {short(kname)}  [{kname[:100]}]")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:62s} {d[k]:>16s} {units[hdr.index(k)]}")
        rd = value(d, units, hdr, "dram__bytes_read.sum")
        wr = value(d, units, hdr, "dram__bytes_write.sum")
        t = value(d, units, hdr, "gpu__time_duration.sum")
        if rd is not None and wr is not None:
            out.append(f"  {'DRAM traffic (read+write)':62s} {rd + wr:16.0f} byte")
            if t:
                out.append(f"  {'DRAM traffic / duration':62s} {(rd + wr) / t / 1e9:16.1f} GB/s")
            # several captured launches of one kernel (e.g. one hook launch per
            # edge window) add up to one ExecStats launch record
            w = traffic.setdefault(workload, {})
            key = short(kname)
            w[key] = int(rd + wr) + (w.get(key, 0) if key in seen else 0)
            seen.add(key)
        stalls = []
        for k in hdr:
            if k.startswith(STALL) and k.endswith(".ratio"):
                try:
                    stalls.append((float(d[k]), k[len(STALL):-len(".ratio")]))
                except ValueError:
                    pass
        for v, k in sorted(stalls, reverse=True)[:6]:
            out.append(f"  stall {k:56s} {v:16.2f} cycles/inst")
        out.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", name + ".txt"), "w") as f:
        f.write("\n".join(out) + "\n")
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(out))


if __name__ == "__main__":
    main()
