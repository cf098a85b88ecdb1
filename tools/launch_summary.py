"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list over the
last K training steps (each step ends with its chain launch: k_chain<1>, the
fused chain + Adam, or k_adam after k_chain when DSG_FUSE_ADAM=0)."""
import collections
import csv
import re
import sys


def main(path, steps):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    seq = []
    for r in rows[start + 1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        ms = v / 1e6 if r[ui] == "ns" else (v / 1e3 if r[ui] in ("us", "usecond") else v)
        seq.append((re.sub(r".*::", "", re.sub(r"\(.*", "", r[ki])), ms))
    ends = [i for i, (n, _) in enumerate(seq) if n in ("k_adam", "k_chain<1>")]
    adam = ends
    win = seq[adam[-steps - 1] + 1:] if len(adam) > steps else seq
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for n, ms in win:
        tot[n] += ms
        cnt[n] += 1
    T = sum(tot.values())
    print(f"kernel time {T / steps:.4f} ms/step over {steps} steps, {len(win) // steps} launches/step")
    print("| kernel | launches/step | us/launch | ms/step | share |\n|---|---|---|---|---|")
    for n, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| {n} | {cnt[n] / steps:g} | {1e3 * v / cnt[n]:.1f} | {v / steps:.4f} | {100 * v / T:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3)
