"""Per-source-line instruction / stall breakdown of an .ncu-rep (sass joined to cuda lines)."""
import collections
import csv
import subprocess
import sys

import os

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
flt = os.environ.get("NCU_FILTER", "").split()   # e.g. "--kernel-name regex:k_seg_spec --launch-skip 1 --launch-count 1"
a = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                   capture_output=True, text=True).stdout.splitlines()
b = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source", "sass"],
                   capture_output=True, text=True).stdout.splitlines()
addr2line, cur, curfile = {}, None, None
for r in csv.reader(a):
    if r and r[0] == "File Path":
        curfile = r[1].split("/")[-1]
    elif len(r) >= 4 and r[0] and r[0] not in ("Line No", "Function Name"):
        cur = (curfile, int(r[0]), r[1].strip()[:80])
    elif len(r) >= 4 and r[2].startswith("0x"):
        addr2line[r[2]] = cur
rows = list(csv.reader(b))
h = rows[1]
ia, ie, iw = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
L, W, ops = collections.Counter(), collections.Counter(), collections.Counter()
tot = tw = 0
for r in rows[2:]:
    if len(r) <= ie:
        continue
    try:
        n, w = int(r[ie]), int(r[iw])
    except ValueError:
        continue
    k = addr2line.get(r[ia])
    L[k] += n
    W[k] += w
    tot += n
    tw += w
    t = r[h.index("Source")].split()
    op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]
    ops[op] += n
print(f"total warp instructions {tot}")
print("ops:", ", ".join(f"{o} {n / tot * 100:.1f}%" for o, n in ops.most_common(12)))
print("-- by instructions")
for k, n in L.most_common(top):
    print(f"{n / tot * 100:5.1f}% inst {W[k] / tw * 100:5.1f}% stall  {k}")
print("-- by stall samples")
for k, n in W.most_common(top):
    print(f"{L[k] / tot * 100:5.1f}% inst {n / tw * 100:5.1f}% stall  {k}")

# optional phase split: --ranges name:lo-hi,name:lo-hi (lines of the main file)
if len(sys.argv) > 3:
    spans = []
    for part in sys.argv[3].split(","):
        name, rng = part.split(":")
        lo, hi = (int(x) for x in rng.split("-"))
        spans.append((name, lo, hi))
    agg_i, agg_w = collections.Counter(), collections.Counter()
    for k in L:
        name = "other"
        if k and k[0] == "mcb_kernels.cu":
            for nm, lo, hi in spans:
                if lo <= k[1] <= hi:
                    name = nm
                    break
        agg_i[name] += L[k]
        agg_w[name] += W[k]
    print("-- by phase")
    for name in [s[0] for s in spans] + ["other"]:
        print(f"{name:10s} {agg_i[name] / tot * 100:5.1f}% inst {agg_w[name] / tw * 100:5.1f}% stall")
