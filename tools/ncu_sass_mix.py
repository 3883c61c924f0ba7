"""Summarise an `ncu --page source --csv` SASS dump: instruction mix and top stall sites.
usage: python tools/ncu_sass_mix.py dump.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr = rows[h]
si, ii = hdr.index("Source"), hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
mix, stall = collections.Counter(), collections.Counter()
lines = []
for r in rows[h + 1:]:
    try:
        n, s = int(r[ii]), int(r[ws])
    except (ValueError, IndexError):
        continue
    op = r[si].split()[0] if r[si].split() else "?"
    if op.startswith("@"):
        op = r[si].split()[1]
    op = op.split(".")[0]
    mix[op] += n
    stall[op] += s
    lines.append((s, n, r[0], r[si].strip()[:90]))
tot, tots = sum(mix.values()), sum(stall.values())
print("warp-instructions executed: %d, stall samples: %d" % (tot, tots))
for op, n in mix.most_common(top):
    print("  %-10s %12d  %5.1f%%   stall %5.1f%%" % (op, n, 100.0 * n / tot, 100.0 * stall[op] / max(1, tots)))
print("top stall sites:")
for s, n, a, src in sorted(lines, reverse=True)[:12]:
    print("  %5.1f%%  %10d  %s" % (100.0 * s / max(1, tots), n, src))
