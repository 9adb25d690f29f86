"""DRAM bytes per step of the K3 / K4 stages from an ncu launch list with
dram__bytes_read.sum / dram__bytes_write.sum (one bench step under ncu):

    python tools/traffic_json.py gpurun_out/traffic_c4.csv c4 > profiles/r2_c4_traffic.json

K3 = the scorer kernels (snapshots, tensor-core or float64 scorer, re-score),
K4 = the replay kernels; bench.py reads the file as roofline.traffic."""
import collections
import csv
import json
import sys

K3 = ("k_tile_summary", "k_snap_scan", "k_score", "k_rescore", "k_prep_tc", "k_wscale", "k_prepare_nets",
      "k_feat_snap", "k_tile_offsets")
K4 = ("k_replay", "k_seg_", "k_wseg_", "k_tseg_", "k_replay_wide", "k_replay_solo", "k_fold")

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
for r in rows[1:]:
    try:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        per[r[ii]]["name"] = r[ki]
    except ValueError:
        pass
out = {"k3": 0.0, "k4": 0.0, "k3_ms": 0.0, "k4_ms": 0.0, "kernels": {}}
unit = 1.0
for d in per.values():
    name = d.get("name", "")
    b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    ms = d.get("gpu__time_duration.sum", 0.0)
    short = name.split("(")[0].split("<")[0].split("::")[-1]
    e = out["kernels"].setdefault(short, {"launches": 0, "bytes": 0.0})
    e["launches"] += 1
    e["bytes"] += b
    if any(name.split("(")[0].find(k) >= 0 for k in K3):
        out["k3"] += b
        out["k3_ms"] += ms
    elif any(name.split("(")[0].find(k) >= 0 for k in K4):
        out["k4"] += b
        out["k4_ms"] += ms
calls = max(1, out["kernels"].get("k_fold", {}).get("launches", 1))   # one k_fold per replay call
for k in ("k3", "k4", "k3_ms", "k4_ms"):
    out[k] /= calls
out["k3_ms"] /= 1e6
out["k4_ms"] /= 1e6
out["calls_under_ncu"] = calls
out["workload"] = sys.argv[2]
out["source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum over one "
                 "bench.py run (--print-units base), divided by the number of replay calls in it: bytes and ms per step")
print(json.dumps(out, indent=1))
