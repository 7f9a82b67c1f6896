"""Summarise an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes]) per kernel name, for the
last decode step and the last correct_kernel of the capture.  usage: launch_summary.py <csv>"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
launch, order = {}, []
for r in rows[start + 1:]:
    lid = int(r[0])
    if lid not in launch:
        launch[lid] = {"name": r[ik].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0].replace("void ", "").replace("sirius::", "").split("<")[0]
                       .replace("(anonymous namespace)::", "")}
        order.append(lid)
    launch[lid][r[im]] = float(r[iv].replace(",", ""))
names = [launch[l]["name"] for l in order]
fin = [i for i, n in enumerate(names) if "accept_finalize" in n]
def seg_summary(title, seg):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for l in seg:
        d = launch[l]; a = agg[d["name"]]
        a[0] += 1; a[1] += d.get("gpu__time_duration.sum", 0); a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    print(f"== {title}: {len(seg)} launches, {tot / 1e3:.1f} us total device time")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = a[2] / a[1] if a[1] else 0
        print(f"   {k:28s} n={a[0]:4d} sum={a[1] / 1e3:9.1f}us avg={a[1] / a[0] / 1e3:8.2f}us  {a[2] / 1e6:9.1f}MB  {gbs:7.1f} GB/s")
# verify segment: from the head gemv before the last accept_finalize
last = fin[-1]
j = last
while j > 0 and names[j] != "gemv_kernel": j -= 1  # the head GEMV of the last draft step
seg_summary("correct_kernel (last)", order[j + 1:last + 1])
# the verify's first layers launch by launch (GEMMs in order: QKV, O, gate+up, down)
print("   first verify launches:", ", ".join(f"{names[i].replace('_kernel', '')} {launch[order[i]].get('gpu__time_duration.sum', 0) / 1e3:.1f}"
                                         for i in range(j + 1, min(j + 18, last + 1))))
# one decode step: the launches between the last two head GEMVs before the verify
heads = [i for i in range(j + 1) if names[i] == "gemv_kernel" and launch[order[i]].get("dram__bytes_read.sum", 0) > 5e8]
if len(heads) >= 2:
    seg_summary("one sparse decode step", order[heads[-2] + 1:heads[-1] + 1])
