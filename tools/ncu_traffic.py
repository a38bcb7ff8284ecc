"""Read an `ncu --set full` report of k_gather and store its DRAM traffic per
launch into profiles/refine_traffic.json under the bench config key."""
import csv
import io
import json
import os
import subprocess
import sys

rep, key = sys.argv[1], sys.argv[2]
# an .ncu-rep, or its `--page raw --csv` export
raw = (open(rep).read() if rep.endswith(".csv") else
       subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
rows = [r for r in csv.reader(io.StringIO(raw)) if r]
while rows and rows[0][0] != "ID":  # ncu banner lines before the header
    rows.pop(0)
hdr = rows[0]
out = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if "k_gather" not in d.get("Kernel Name", ""):
        continue
    unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    rd = float(d["dram__bytes_read.sum"].replace(",", "")) * unit.get(rows[1][hdr.index("dram__bytes_read.sum")], 1)
    wr = float(d["dram__bytes_write.sum"].replace(",", "")) * unit.get(rows[1][hdr.index("dram__bytes_write.sum")], 1)
    out = {"dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
           "l2_hit_pct": float(d["lts__t_sector_hit_rate.pct"]),
           "duration_ms_under_ncu": float(d["gpu__time_duration.sum"].replace(",", "")) *
           {"msecond": 1.0, "usecond": 1e-3, "second": 1e3}.get(rows[1][hdr.index("gpu__time_duration.sum")], 1.0),
           "dram_throughput_pct": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
           "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
           "registers": int(float(d["launch__registers_per_thread"])), "source": os.path.basename(rep)}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "refine_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
db[key] = out
json.dump(db, open(path, "w"), indent=1)
print(key, json.dumps(out))
