"""Print the hottest SASS lines (warp-stall samples) of one kernel in an .ncu-rep."""
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
si = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source"); ie = h.index("Instructions Executed")
num = lambda v: int(float(v)) if v.strip().replace(".", "", 1).isdigit() else 0
tot = sum(num(x[si]) for x in rows)
print("samples", tot, "instructions", sum(num(x[ie]) for x in rows))
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
agg = {h[i]: sum(num(x[i]) for x in rows) for i in stall_cols}
print("stalls:", sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:8])
for x in sorted(rows, key=lambda x: -num(x[si]))[:n]:
    print(f"{num(x[si]):6d} {num(x[ie]):9d}  {x[src][:100]}")
