"""Print the hottest SASS lines (warp-stall samples) of an ncu report: ncu_hot.py <rep> [n]."""
import csv, subprocess, sys, io
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
kernels = []
cur = None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; kernels.append(cur)
    elif cur is not None:
        cur.append(ln)
for k in kernels[:1]:
    rows = list(csv.reader(io.StringIO("\n".join(k[1:]))))
    hdr = rows[0]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_e = hdr.index("Instructions Executed")
    tot = sum(float(r[i_s] or 0) for r in rows[1:])
    print(k[0][:150], "total samples", tot)
    for r in sorted(rows[1:], key=lambda r: -float(r[i_s] or 0))[:n]:
        print(f"{float(r[i_s]) / tot * 100:5.1f}%  exec {r[i_e]:>8}  {r[0][-5:]} {r[1].strip()[:100]}")
