"""Summarise ncu reports into profiles/: per-kernel key counters (text + JSON)."""
import csv
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_shared_mem", "occ_limit_smem_blocks"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall_short_sb"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_barrier"),
]


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit)
    return float(v.replace(",", "")) * mult if mult else None


def main(rep, out_txt, out_json):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                val, unit = r[i], u[i]
                if unit in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                    d[name + "_bytes"] = to_bytes(val, unit)
                elif k == "gpu__time_duration.sum":
                    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1.0)
                    d["duration_ms"] = float(val.replace(",", "")) * scale
                else:
                    try:
                        d[name] = float(val.replace(",", ""))
                    except ValueError:
                        d[name] = val
        if "dram_read_bytes" in d:
            d["dram_traffic_bytes"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0.0)
        res.append(d)
    with open(out_json, "w") as f:
        json.dump(res, f, indent=1)
    with open(out_txt, "w") as f:
        for d in res:
            f.write(f"== {d['kernel']}\n")
            for k, v in d.items():
                if k != "kernel":
                    f.write(f"  {k:28s} {v}\n")
    print(open(out_txt).read())


if __name__ == "__main__":
    main(*sys.argv[1:4])
