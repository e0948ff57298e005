"""Top stalled SASS instructions and stall-reason totals of one launch in an ncu report.
usage: python tools/ncu_stalls.py REP [launch_index] [top]"""
import csv
import subprocess
import sys


def main(rep, idx=0, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    si = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")
    stall_cols = [(c, i) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = {c: 0 for c, _ in stall_cols}
    data = []
    for k, r in enumerate(rows[hi + 1:]):
        try:
            v = int(r[si])
        except (ValueError, IndexError):
            continue
        for c, i in stall_cols:
            try:
                tot[c] += int(r[i])
            except ValueError:
                pass
        reasons = sorted(((int(r[i]) if r[i].isdigit() else 0, c[6:]) for c, i in stall_cols), reverse=True)[:2]
        data.append((v, k, r[src][:70], reasons))
    allv = sum(d[0] for d in data)
    print("samples", allv, "| reasons:", ", ".join(f"{c[6:]}={v}" for c, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
    for d in sorted(data, reverse=True)[:top]:
        print(f"{d[0]:6d} #{d[1]:5d} {d[2]:70s} {d[3]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 25)
