"""Hottest SASS instructions of one kernel with their top stall reasons, plus
shared-memory wavefront totals.  usage: ncu_hot.py report kernel-regex [n]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source=sass"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]; rows = []
for x in r[2:]:
    if x and x[0] == "Kernel Name":
        break
    if len(x) == len(h) and x[0] != "Address":
        rows.append(x)
def num(v):
    try: return float(v)
    except: return 0.0
si = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source"); ie = h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(num(x[si]) for x in rows)
print("samples", tot, "instructions", sum(num(x[ie]) for x in rows))
agg = {h[i]: sum(num(x[i]) for x in rows) for i in stall_cols}
print("stalls:", [(k[6:], int(v)) for v, k in sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:8]])
for name in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal"):
    if name in h:
        print(name, sum(num(x[h.index(name)]) for x in rows))
for x in sorted(rows, key=lambda x: -num(x[si]))[:n]:
    st = sorted(((num(x[i]), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    print(f"{num(x[si]):6.0f} {num(x[ie]):9.0f}  {x[src][:60]:60s} {st[0][1]}:{st[0][0]:.0f} {st[1][1]}:{st[1][0]:.0f}")
