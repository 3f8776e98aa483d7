"""Key metrics of each kernel in an ncu report (details page)."""
import csv, subprocess, sys
want = ['Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Executed Ipc Active',
        'Issue Slots Busy', 'Dynamic Shared Memory Per Block', 'Block Size', 'Grid Size',
        'DRAM Throughput', 'Warp Cycles Per Issued Instruction', 'Theoretical Occupancy',
        'Compute (SM) Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate']
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'details', '--csv'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
seen = set()
for r in rows[1:]:
    key = (r[ki][:30], r[mi])
    if r[mi] in want and key not in seen:
        seen.add(key)
        print(r[ki].split('(')[0][-24:].ljust(24), r[mi].ljust(36), r[vi], r[ui])
