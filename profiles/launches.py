"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel
for the last complete wave(s). Usage: python profiles/launches.py <csv> [waves]"""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, mi, vi, ii = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'ID'))
    per, names = collections.defaultdict(dict), {}
    for r in data:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(',', ''))
        names[int(r[ii])] = r[ki]
    return per, names


def short(n):
    m = re.search(r'(k_\w+)(<[^(]*>)?', n)
    return (m.group(1) + (m.group(2) or '')) if m else n[:40]


def main():
    per, names = load(sys.argv[1])
    waves = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    ids = sorted(per)
    # wave starts (k_prepare) that are followed by a gather before the next
    # wave: the bench's own waves, not the device simulate() of the alpha
    # sweep the bench runs after its timed regions
    starts = [i for i in ids if short(names[i]) == 'k_prepare']
    bounds = starts + [ids[-1] + 1]
    starts = [a for a, b in zip(bounds, bounds[1:])
              if any(re.match(r'k_gather(<|$)', short(names[j])) for j in ids if a <= j < b)]
    lo = starts[-waves]
    nxt = next((b for b in bounds if b > starts[-1]), ids[-1] + 1)
    hi = max(j for j in ids if starts[-1] <= j < nxt and re.match(r'k_gather(<|$)', short(names[j]))) + 1
    # the wave's own kernels only: torch kernels the bench runs after the timed
    # regions (distinct-row count, tallies) are not part of a wave
    sel = [i for i in ids if lo <= i < hi and not re.search(r'at_cuda_detail|at::', names[i])]
    agg = collections.OrderedDict()
    for i in sel:
        k = short(names[i])
        a = agg.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += per[i].get('gpu__time_duration.sum', 0)
        a[2] += per[i].get('dram__bytes_read.sum', 0) + per[i].get('dram__bytes_write.sum', 0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':34s} {'launches':>8s} {'us/wave':>10s} {'share':>7s} {'DRAM MB/wave':>13s}")
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:34s} {c // waves:8d} {t / 1e3 / waves:10.1f} {100 * t / tot:6.1f}% {b / waves / 1e6:13.1f}")
    print(f"{'total':34s} {'':8s} {tot / 1e3 / waves:10.1f}")


if __name__ == '__main__':
    main()
