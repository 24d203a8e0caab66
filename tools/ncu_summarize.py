"""Summarise ncu outputs into the committed profiles/ tables (diagnostics).

  python tools/ncu_summarize.py launches <ncu --csv launch list> <out.csv>
      one row per kernel launch: idx, kernel, gpu_time_us (ncu --metrics gpu__time_duration.sum,
      serialised and cold-cache: compare shares, not absolutes)
  python tools/ncu_summarize.py full <report.ncu-rep> <out.csv>
      per-launch key metrics of an `ncu --set full` capture (dram bytes, DRAM / tensor-pipe
      utilisation, warps active, registers, shared memory)
"""
import csv
import io
import subprocess
import sys


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
    gi, bi = hdr.index("Grid Size"), hdr.index("Block Size")
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["idx", "kernel", "grid", "block", "gpu_time_us"])
        for r in rows[h + 1:]:
            w.writerow([r[ii], r[ki].split("(")[0], r[gi], r[bi], f"{float(r[vi]) / 1e3:.2f}"])


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__shared_mem_per_block_dynamic"]


def full(rep, dst):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    cols = [hdr.index(m) for m in METRICS if m in hdr]
    ki, gi = hdr.index("Kernel Name"), hdr.index("Grid Size")
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["Kernel Name", "Grid Size"] + [f"{hdr[c]} [{units[c]}]" for c in cols])
        for r in rows[2:]:
            w.writerow([r[ki], r[gi]] + [r[c] for c in cols])


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
