"""Summarise one ncu --set full capture: headline metrics, opcode mix
(instructions per element) and the hottest stall lines.

    python tools/ncu_summary.py gpurun_out/prof_apply_v6.ncu-rep [elements]
    LOPT_NCU_KERNEL=apply_tc python tools/ncu_summary.py <multi-kernel report>
"""
import collections
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
elems = float(sys.argv[2]) if len(sys.argv) > 2 else 86567656.0
# LOPT_NCU_KERNEL=regex selects one kernel of a multi-kernel report
KF = ['-k', 'regex:' + os.environ['LOPT_NCU_KERNEL']] if os.environ.get('LOPT_NCU_KERNEL') else []
want = ['Duration', 'DRAM Throughput', 'Executed Ipc Active', 'Issue Slots Busy', 'No Eligible',
        'Active Warps Per Scheduler', 'Eligible Warps Per Scheduler',
        'Warp Cycles Per Issued Instruction', 'Issued Instructions', 'Registers Per Thread',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'SM Frequency']
det = subprocess.run(['ncu', '-i', rep] + KF + [ '--page', 'details', '--csv'], capture_output=True, text=True).stdout
for r in csv.reader(io.StringIO(det)):
    if len(r) > 14 and r[12] in want:
        print(f"{r[12]:40s} {r[14]} {r[13]}")
raw = subprocess.run(['ncu', '-i', rep] + KF + [ '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
if len(rows) > 2:
    hdr, units, vals = rows[0], rows[1], rows[2]
    for key in ('dram__bytes_read.sum', 'dram__bytes_write.sum'):
        if key in hdr:
            i = hdr.index(key)
            print(f"{key:40s} {vals[i]} {units[i]}")
src = subprocess.run(['ncu', '-i', rep] + KF + [ '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
tot = sum(int(r[iE]) for r in data)
stall = sum(int(r[iS]) for r in data) or 1
print(f"warp instructions per element: {tot / elems * 32:.1f} thread-instr (all warps)")
h = collections.Counter()
hs = collections.Counter()
for r in data:
    t = r[1].split()
    op = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
    h[op] += int(r[iE])
    hs[op] += int(r[iS])
print("opcode      per-elem  stall%")
for op, c in h.most_common(30):
    print(f"{op:12s} {c / elems * 32:8.1f} {100 * hs[op] / stall:6.1f}")
print("hottest stall lines:")
idx = sorted(range(len(data)), key=lambda i: -int(data[i][iS]))[:12]
for i in sorted(idx):
    print(f"  {i:5d} {100 * int(data[i][iS]) / stall:5.1f}%  {data[i][1][:80]}")
    for k in range(max(0, i - 3), i):
        print(f"        {data[k][1][:80]}")
