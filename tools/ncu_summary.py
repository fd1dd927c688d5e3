"""One-line-per-metric summary of ncu --page details/raw csv dumps:
python tools/ncu_summary.py <prefix> ...  (reads <prefix>.details.csv, <prefix>.raw.csv)"""
import csv
import sys

WANT = ["Duration", "Compute (SM) Throughput", "DRAM Throughput", "Memory Throughput",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Issue Slots Busy",
        "Executed Ipc Active", "L2 Hit Rate", "Waves Per SM", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block"]
RAW = ["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "dram__bytes_read.sum", "dram__bytes_write.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
       "smsp__inst_executed.sum"]
for k in sys.argv[1:]:
    print("=====", k)
    rows = list(csv.reader(open(f"{k}.details.csv")))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    seen = set()
    for r in rows[1:]:
        name = r[idx["Metric Name"]]
        if name in WANT and name not in seen:
            seen.add(name)
            print(f"  {name}: {r[idx['Metric Value']]} {r[idx['Metric Unit']]}")
    raw = list(csv.reader(open(f"{k}.raw.csv")))
    h, u, v = raw[0], raw[1], raw[2]
    for i, name in enumerate(h):
        if name in RAW:
            print(f"   {name}: {v[i]} {u[i]}")
