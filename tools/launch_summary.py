"""Per-kernel summary of an ncu launch list (CSV written by
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
      --clock-control none --csv --log-file LIST.csv python bench.py --steps S --warmup W)
as the per-step traffic JSON bench.py reads (profiles/r02_traffic_cfg5.json) and a text table.
python tools/launch_summary.py LIST.csv STEPS_TOTAL OUT.json [OUT.txt]
STEPS_TOTAL = steps + warmup of the profiled command (per-step figures = totals / STEPS_TOTAL)."""
import csv
import json
import re
import sys

path, nsteps, out_json = sys.argv[1], int(sys.argv[2]), sys.argv[3]
out_txt = sys.argv[4] if len(sys.argv) > 4 else None
rows = []
with open(path, newline="") as f:
    lines = [l for l in f if l.startswith('"')]
rd = csv.DictReader(lines)
per = {}
conv = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
for r in rd:
    name = r["Kernel Name"]
    m = re.search(r"(?:cs::(?:tcb::)?)?(\w+)(?:<|\()", name.replace("void ", ""))
    short = m.group(1) if m else name
    d = per.setdefault(short, {"ids": set(), "time_ms": 0.0, "rd": 0.0, "wr": 0.0})
    d["ids"].add(r["ID"])
    v = float(r["Metric Value"].replace(",", "")) * conv.get(r["Metric Unit"], 1.0)
    if r["Metric Name"] == "gpu__time_duration.sum":
        d["time_ms"] += v
    elif r["Metric Name"] == "dram__bytes_read.sum":
        d["rd"] += v
    elif r["Metric Name"] == "dram__bytes_write.sum":
        d["wr"] += v
tot = sum(d["time_ms"] for d in per.values())
res = {"source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum over the bench command "
                 f"({path}), divided by {nsteps} steps", "per_step": {}}
table = []
for k, d in sorted(per.items(), key=lambda kv: -kv[1]["time_ms"]):
    e = {"launches": len(d["ids"]) / nsteps, "time_ms": d["time_ms"] / nsteps, "share": d["time_ms"] / tot,
         "dram_read_GB": d["rd"] / nsteps / 1e9, "dram_write_GB": d["wr"] / nsteps / 1e9}
    res["per_step"][k] = e
    table.append(f"{k:34s} {e['launches']:6.1f}/step {e['time_ms']:10.2f} ms/step {100 * e['share']:5.1f}%  "
                 f"dram rd {e['dram_read_GB']:8.2f} GB wr {e['dram_write_GB']:8.2f} GB")
with open(out_json, "w") as f:
    json.dump(res, f, indent=1)
txt = "\n".join(table)
print(txt)
if out_txt:
    with open(out_txt, "w") as f:
        f.write(txt + "\n")
