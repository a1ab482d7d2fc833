"""Summarise ncu captures for profiles/: per-kernel duration (ms), DRAM traffic (GB, TB/s, % of peak),
pipe utilisation, stalls.
usage: python tools/ncu_summary.py <report.ncu-rep> [...] > profiles/<name>.md"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("time_ms", "gpu__time_duration.sum"),
    ("dram_rd_GB", "dram__bytes_read.sum"),
    ("dram_wr_GB", "dram__bytes_write.sum"),
    ("dram_TB/s", "dram__bytes.sum.per_second"),
    ("dram_%peak", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("dmma_%", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("fp64_%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("warps_%", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("smem_conf", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("st_long", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
    ("st_short", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"),
    ("st_mathpipe", "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"),
    ("st_wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"),
    ("st_barrier", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    # normalise units: time -> ms, bytes -> GB, rates -> TB/s (ncu picks its own prefixes per value)
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
             "byte/second": 1e-12, "Kbyte/second": 1e-9, "Mbyte/second": 1e-6, "Gbyte/s": 1e-3,
             "Gbyte/second": 1e-3, "Tbyte/s": 1.0, "Tbyte/second": 1.0}
    for row in r[2:]:
        d = {"name": row[hdr.index("Kernel Name")]}
        for k, m in KEYS:
            if m not in hdr:
                d[k] = ""
                continue
            i = hdr.index(m)
            v = row[i].replace(",", "")
            try:
                d[k] = str(float(v) * scale.get(units[i], 1.0))
            except ValueError:
                d[k] = v
        yield d


def main():
    print("| kernel | " + " | ".join(k for k, _ in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for rep in sys.argv[1:]:
        for d in rows(rep):
            name = d["name"].replace("void ", "").split("(")[0][:48]
            vals = []
            for k, _ in KEYS:
                v = d[k].replace(",", "")
                try:
                    f = float(v)
                    vals.append(f"{f:.3g}")
                except ValueError:
                    vals.append(v)
            print(f"| {name} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
