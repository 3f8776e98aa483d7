"""Round summary of an `ncu --set full` capture: key details-page metrics plus
per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and
pipe utilisation from the raw page.  Usage: ncu_full_summary.py REPORT..."""
import csv
import subprocess
import sys

DETAILS = ['Duration', 'Registers Per Thread', 'Block Size', 'Grid Size', 'Dynamic Shared Memory Per Block',
           'Achieved Occupancy', 'Executed Ipc Active', 'Issue Slots Busy', 'Warp Cycles Per Issued Instruction',
           'Compute (SM) Throughput', 'Memory Throughput', 'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate']
RAW = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
       'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
       'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
       'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
       'smsp__inst_executed.sum', 'sm__cycles_elapsed.max']


def run(rep, page):
    out = subprocess.run(['ncu', '-i', rep, '--page', page, '--csv'], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


for rep in sys.argv[1:]:
    rows = run(rep, 'details')
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
    name = rows[1][ki].split('(')[0]
    print(f"== {name}  ({rep.split('/')[-1]})")
    seen = set()
    for r in rows[1:]:
        if r[mi] in DETAILS and r[mi] not in seen:
            seen.add(r[mi])
            print(f"   {r[mi]:40s} {r[vi]} {r[ui]}")
    raw = run(rep, 'raw')
    hdr, units, vals = raw[0], raw[1], raw[2]
    for m in RAW:
        if m in hdr:
            i = hdr.index(m)
            print(f"   {m:60s} {vals[i]} {units[i]}")
    if 'dram__bytes_read.sum' in hdr:
        def b(m):
            i = hdr.index(m)
            v = float(vals[i].replace(',', ''))
            u = units[i]
            return v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
        print(f"   traffic (dram read+write) per launch      {b('dram__bytes_read.sum') + b('dram__bytes_write.sum'):.0f} bytes")
