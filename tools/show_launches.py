import csv, sys
lines = open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv').read().splitlines()
i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
tot = 0
for r in csv.DictReader(lines[i:]):
    if r['Metric Name'] != 'gpu__time_duration.sum': continue
    v = float(r['Metric Value']) / 1000; tot += v
    print(f"{r['Kernel Name'][:60]:60s} {r['Grid Size']:>14s} {v:8.1f} us")
print(f"total {tot:.1f} us")
