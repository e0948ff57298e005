"""Summarise an ncu report: per launch key metrics (duration, DRAM bytes, throughput, occupancy)."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "launch__grid_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "smsp__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tensor.sum"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki = h.index("Kernel Name")
    cols = [(w, h.index(w)) for w in WANT if w in h]
    for r in rows[2:]:
        print(r[ki][:70])
        print("   " + ", ".join(f"{w.split('.')[0].replace('__', ':')}{'.' + w.split('.')[-1] if 'pct' in w else ''}={r[i]}" for w, i in cols))


if __name__ == "__main__":
    main(sys.argv[1])
