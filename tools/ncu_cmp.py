"""Side-by-side key metrics of `ncu --page raw --csv` exports (one row per kernel launch).
usage: python tools/ncu_cmp.py a.csv b.csv ...   (metric-name substrings via -m a,b,c)"""
import csv
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum", "smsp__sass_inst_executed_op_utcmma.sum"]
args = [a for a in sys.argv[1:] if not a.startswith("-m")]
for a in sys.argv[1:]:
    if a.startswith("-m"):
        KEYS += a[2:].split(",")
for f in args:
    rows = list(csv.reader(open(f)))
    i0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, units = rows[i0], rows[i0 + 1]
    print("==", f)
    for r in rows[i0 + 2:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        print("  " + d.get("Kernel Name", "?")[:60])
        for k in KEYS[1:]:
            for hk in h:
                if hk == k:
                    print("     %-72s %s %s" % (k, d[hk], units[h.index(hk)]))
