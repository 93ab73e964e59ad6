"""Write profiles/traffic_<cfg>.json from one `ncu --set full` capture of k_lanes:
dram__bytes_read.sum + dram__bytes_write.sum of that launch divided by the
lane-cycles it simulated (bench.py scales it back to its own launch).

    python tools/ncu_traffic.py REPORT.ncu-rep CONFIG LANES CYCLES [KERNEL]
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, cfg, lanes, cycles = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
kernel = sys.argv[5] if len(sys.argv) > 5 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def num(k):
    v, u = d[k]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return float(v.replace(",", "")) * scale


rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
out = {"report": os.path.basename(rep), "config": cfg, "lanes": lanes, "cycles": cycles, "kernel": kernel,
       "dram_bytes_read": rd, "dram_bytes_write": wr,
       "dram_bytes_per_lane_cycle": (rd + wr) / (lanes * cycles),
       "gpu_time_ms": float(d["gpu__time_duration.sum"][0].replace(",", "")) *
                      {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(
                          d["gpu__time_duration.sum"][1], float("nan")),
       "note": "ncu --set full --clock-control none (cache control all: caches flushed before the captured launch)"}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    os.environ.get("RS_PROFILE_ROUND", "r02"), f"traffic_{cfg}.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out))
