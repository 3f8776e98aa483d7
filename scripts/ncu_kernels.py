"""Per-kernel summary of a multi-kernel `ncu --set full` report: duration,
DRAM traffic (read + write), pipe utilisation, IPC, occupancy."""
import csv
import subprocess
import sys

M = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
     'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
     'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
     'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
     'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
     'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
     'sm__instruction_throughput.avg.pct_of_peak_sustained_active']
for rep in sys.argv[1:]:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    idx = {m: h.index(m) for m in M if m in h}
    scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-3, 'usecond': 1.0, 'ns': 1e-3, 'us': 1.0, 'ms': 1e3,
             'msecond': 1e3, 'second': 1e6}
    ki = h.index('Kernel Name')
    print(f"== {rep}")
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        name = r[ki].split('(')[0].replace('<unnamed>::', '').replace('void ', '')[:44]
        v = {m: r[i].replace(',', '') for m, i in idx.items()}
        sc = {m: scale.get(units[i], 1.0) for m, i in idx.items()}
        dur = float(v['gpu__time_duration.sum']) * sc['gpu__time_duration.sum']
        rd = float(v['dram__bytes_read.sum']) * sc['dram__bytes_read.sum']
        wr = float(v['dram__bytes_write.sum']) * sc['dram__bytes_write.sum']
        print(f"{name:44s} dur {dur:10.1f} us | dram {rd + wr:14.0f} B (r {rd:.3g} w {wr:.3g}) | "
              f"fp64 {float(v[M[3]]):5.1f}% tensor {float(v[M[4]]):5.1f}% fma {float(v[M[5]]):5.1f}% "
              f"lsu {float(v[M[6]]):5.1f}% | warps {float(v[M[8]]):5.1f}% | inst {float(v[M[7]]):.3g}")
