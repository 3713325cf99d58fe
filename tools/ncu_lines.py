"""Aggregate ncu source metrics per CUDA source line (cuda,sass view) for one kernel.
usage: ncu_lines.py report.ncu-rep kernel-regex [n] [sort: samples|instr]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
key = 1 if (len(sys.argv) > 4 and sys.argv[4] == "instr") else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
def num(v):
    try: return float(v)
    except: return 0.0
rows = []; fname = "?"; h = None
for x in csv.reader(out.splitlines()):
    if not x: continue
    if x[0] == "File Path": fname = x[1].split("/")[-1]; continue
    if x[0] == "Function Name": continue
    if x[0] == "Line No": h = x; continue
    if h and x[0]:
        rows.append((fname, x))
si = h.index("Warp Stall Sampling (All Samples)"); ie = h.index("Instructions Executed")
agg = {}
for f, x in rows:
    k = (f, x[0], x[1].strip()[:80])
    a = agg.setdefault(k, [0, 0]); a[0] += num(x[si]); a[1] += num(x[ie])
tot = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
print(f"samples {tot:.0f} warp-instructions {ti:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:n]:
    print(f"{v[0]:7.0f} {v[1]:11.0f}  {k[0]}:{k[1]:<4} {k[2]}")
