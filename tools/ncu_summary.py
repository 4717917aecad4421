"""Compact summary of ncu reports (key throughput / DRAM metrics per launch).
usage: python tools/ncu_summary.py out.csv rep1.ncu-rep [rep2 ...]"""
import csv, subprocess, sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__issue_inst0.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(h, row))
        yield d.get("Kernel Name", "?"), {k: d.get(k, "") for k in KEYS}, dict(zip(h, units))


def main():
    dst = sys.argv[1]
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["report", "kernel"] + KEYS)
        first = True
        for rep in sys.argv[2:]:
            for name, vals, units in rows(rep):
                if first:
                    w.writerow(["(units)", ""] + [units.get(k, "") for k in KEYS])
                    first = False
                w.writerow([rep.split("/")[-1], name[:90]] + [vals[k] for k in KEYS])
    print(open(dst).read())


if __name__ == "__main__":
    main()
