"""Attribute ncu per-SASS-instruction counts to CUDA source lines.

usage: python tools/ncu_lines.py report.ncu-rep kernel_regex mangled_name [top]
  runs `ncu --page source --csv` for the kernel, `nvdisasm -g` on libbnn.so's sm_100a cubin, maps
  each SASS offset to its //## File/line annotation and prints the hottest lines by executed warp
  instructions and by stall samples.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, kre, mangled = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    hdr = rows[h]
    ai, ii = hdr.index("Address"), hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    recs = []
    for r in rows[h + 1:]:
        try:
            recs.append((int(r[ai], 16), int(r[ii]), int(r[si])))
        except (ValueError, IndexError):
            break  # first kernel instance only
    base = recs[0][0]
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1808_00209_b200", "libbnn.so")], cwd=tmp,
                   capture_output=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
    lines = dis.splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith(".text." + mangled + ":"))
    end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//-----")), len(lines))
    line_of, cur = {}, "?"
    for ln in lines[start:end]:
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = "%s:%s" % (os.path.basename(m.group(1)), m.group(2))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            line_of[int(m.group(1), 16)] = cur
    by_n, by_s = collections.Counter(), collections.Counter()
    for a, n, s in recs:
        key = line_of.get(a - base, "?")
        by_n[key] += n
        by_s[key] += s
    tn, ts = sum(by_n.values()), max(1, sum(by_s.values()))
    print("warp-instructions %d, stall samples %d" % (tn, ts))
    print("%-28s %14s %7s %7s" % ("line", "instr", "%instr", "%stall"))
    for key, n in by_n.most_common(top):
        print("%-28s %14d %6.1f%% %6.1f%%" % (key, n, 100.0 * n / tn, 100.0 * by_s[key] / ts))


if __name__ == "__main__":
    main()
