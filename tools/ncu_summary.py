"""Summarise an ncu --set full report: per kernel launch, the roofline inputs
(duration, DRAM bytes, throughput %, smem wavefronts vs ideal, issue/warps
active).  Also writes profiles/traffic.json (DRAM bytes per launch per
operator kernel) for bench.py's roofline.traffic field.
usage: ncu_summary.py report.ncu-rep out.txt [workload]
traffic.json is stamped with the source hash of libibcuda.so
(_build.source_id: sources, C ABI header, nvcc flags -- summarise before
editing them) and the bench workload, so bench.py only reports it for the
same code."""
import csv, json, subprocess, sys
from pathlib import Path
rep, outp = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
want = [("gpu__time_duration.sum", "duration_us", 1e-3), ("dram__bytes_read.sum", "dram_read_MB", 1e-6),
        ("dram__bytes_write.sum", "dram_write_MB", 1e-6),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct", 1),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts", 1),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct", 1),
        ("launch__registers_per_thread", "regs", 1), ("launch__grid_size", "grid", 1),
        ("smsp__inst_executed.sum", "warp_instructions", 1)]
units = r[1]
lines, traffic = [], {}
for row in r[2:]:
    name = row[h.index("Kernel Name")]
    d = {}
    for key, label, scale in want:
        if key in h:
            v = row[h.index(key)].replace(",", "")
            try:
                val = float(v)
                u = units[h.index(key)]
                if key.startswith("dram__bytes"):
                    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    val = val * mult * scale
                elif key == "gpu__time_duration.sum":
                    mult = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)
                    val = val * mult * scale
                else:
                    val *= scale
                d[label] = round(val, 3)
            except ValueError:
                pass
    lines.append(f"{name[:70]}\n    " + "  ".join(f"{k}={v}" for k, v in d.items()))
    total = (d.get("dram_read_MB", 0) + d.get("dram_write_MB", 0)) * 1e6
    for tag, key in (("spread", "spread_banks"), ("interp", "interp_tma")):
        if key in name:
            traffic[tag] = int(total)
Path(outp).write_text("\n".join(lines) + "\n")
if traffic:
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2012_06646_b200 import _build
    traffic["build"] = _build.source_id()  # the sources the capture's build came from
    traffic["workload"] = sys.argv[3] if len(sys.argv) > 3 else "c2"
    Path("profiles/traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print("\n".join(lines))
