"""Per-kernel shares of the DELTA step in an ncu launch list (the --metrics gpu__time_duration
pass over `bench.py --steps 2`): finds the windows of consecutive launches that form one DELTA
step (35 launches at C1: 32 attention + 3 select) and sums durations by kernel.
usage: python tools/launch_shares.py launches.csv [launches_per_step]"""
import collections
import csv
import sys


def main(path, per_step=35):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    seq = []
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            seq.append((r[ki].split("(")[0].replace("void ", "").replace("delta::<unnamed>::", ""),
                        float(r[vi].replace(",", "")) / 1e3))
    is_step = lambda n: n.startswith(("attn_tc_kernel", "sparse_lat_kernel", "select_kernel"))
    steps, i = [], 0
    while i + per_step <= len(seq):
        w = seq[i:i + per_step]
        if all(is_step(n) for n, _ in w) and sum(n.startswith("select") for n, _ in w) == 3 and \
                sum(n.startswith("sparse_lat") for n, _ in w) >= 20:
            steps.append(w)
            i += per_step
        else:
            i += 1
    tot, cnt = collections.Counter(), collections.Counter()
    for w in steps:
        for n, d in w:
            tot[n] += d
            cnt[n] += 1
    s = sum(tot.values())
    print(f"{len(steps)} DELTA steps found ({per_step} launches each); serialized, cold-cache ncu durations")
    for n, v in tot.most_common():
        print(f"  {n:48s} launches/step {cnt[n] / max(1, len(steps)):5.1f}  mean {v / cnt[n]:7.2f} us  share {v / s:.3f}")
    print(f"  step sum {s / max(1, len(steps)):.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 35)
