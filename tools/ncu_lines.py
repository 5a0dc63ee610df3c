"""Attribute one ncu capture's executed instructions to CUDA source lines.

    python tools/ncu_lines.py <report.ncu-rep> <object.o> <mangled kernel> [elements] [top]
    (LOPT_NCU_KERNEL=regex selects one kernel of a multi-kernel report)

The SASS page of the report gives executed warp-instructions per address; the
object's cubin, disassembled with line info (nvdisasm -g), maps each offset to
its source line.  Prints thread-instructions per element per source line
(inlined helpers appear under their own file:line), hottest first, and the
same totals per opcode within each line.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, fun = sys.argv[1:4]
elems = float(sys.argv[4]) if len(sys.argv) > 4 else 86567656.0
top = int(sys.argv[5]) if len(sys.argv) > 5 else 60

KF = ['-k', 'regex:' + os.environ['LOPT_NCU_KERNEL']] if os.environ.get('LOPT_NCU_KERNEL') else []
src = subprocess.run(['ncu', '-i', rep] + KF + ['--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
iE = hdr.index("Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [(i, h[len("stall_"):]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][0], 16)
execd = {int(r[0], 16) - base: (int(r[iE]), int(r[iS]), r[1].strip()) for r in data}
why = {int(r[0], 16) - base: {nm: int(r[i] or 0) for i, nm in reasons} for r in data}

tmp = tempfile.mkdtemp()
subprocess.run(['cuobjdump', '-xelf', 'all', os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith('.cubin')][0]
dis = subprocess.run(['nvdisasm', '-g', '-c', os.path.join(tmp, cub)], capture_output=True, text=True).stdout
lines = dis.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(fun + ':'))
loc = '?'
amap = {}
for l in lines[start + 1:]:
    if l.startswith('.text.') or l.startswith('\t.section'):
        if amap:
            break
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        loc = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r'\s+/\*([0-9a-f]+)\*/', l)
    if m:
        amap[int(m.group(1), 16)] = loc
    if l.startswith('//---') and amap:
        break

per = collections.Counter()
stl = collections.Counter()
ops = collections.defaultdict(collections.Counter)
rsn = collections.defaultdict(collections.Counter)
tot = 0
for a, (n, s, txt) in execd.items():
    where = amap.get(a, '?')
    per[where] += n
    stl[where] += s
    t = txt.split()
    op = (t[1] if t and t[0].startswith('@') else (t[0] if t else '?')).split('.')[0]
    ops[where][op] += n
    rsn[where].update(why[a])
    tot += n
stot = sum(stl.values()) or 1
print(f"total {tot / elems * 32:.1f} thread-instr/element")
for where, n in per.most_common(top):
    mix = ' '.join(f"{o}:{c / elems * 32:.1f}" for o, c in ops[where].most_common(5))
    rs = ' '.join(f"{k}:{100 * c / stot:.1f}" for k, c in rsn[where].most_common(3) if c)
    print(f"{where:28s} {n / elems * 32:7.1f}  stall {100 * stl[where] / stot:5.1f}%  {mix}  [{rs}]")
if os.environ.get("BY_STALL"):
    print("--- by stall samples")
    for where, c in stl.most_common(25):
        rs = ' '.join(f"{k}:{100 * v / stot:.1f}" for k, v in rsn[where].most_common(4) if v)
        print(f"{where:28s} {100 * c / stot:5.1f}%  {per[where] / elems * 32:7.1f} instr  [{rs}]")
