"""Per-kernel launch counts, mean durations and shares from an ncu launch list
(ncu --metrics gpu__time_duration.sum --csv --log-file ...).

    python tools/launch_summary.py gpurun_out/launches_r1.csv
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
im = hdr.index("Metric Name")
tot = collections.OrderedDict()
cnt = collections.Counter()
byt = collections.Counter()
for r in rows[1:]:
    if not r[ik].startswith(("lopt", "void lopt")):
        continue
    if r[im].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[iu], 1)
        byt[r[ik].split("(")[0]] += float(r[iv].replace(",", "")) * scale
        continue
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    v = v / 1e3 if r[iu] in ("ns", "nsecond") else (v * 1e3 if r[iu] in ("ms", "msecond") else v)   # -> us
    name = r[ik].split("(")[0]
    tot[name] = tot.get(name, 0.0) + v
    cnt[name] += 1
s = sum(tot.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialized): "
      "per-kernel shares of the lopt kernels in the run")
for k, v in tot.items():
    extra = f" dram_MB/launch={byt[k] / cnt[k] / 1e6:8.1f}" if byt else ""
    print(f"{k:55s} launches={cnt[k]:3d} avg_us={v / cnt[k]:9.1f} share={100 * v / s:5.1f}%{extra}")
if byt:
    print(f"all lopt kernels: {sum(byt.values()) / max(cnt.values()) / 1e9:.3f} GB DRAM per step")
