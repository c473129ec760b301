"""Per-instruction stall attribution from an ncu report's SASS source page.

  python tools/ncu_stalls.py report.ncu-rep [--top 40] [--range 0x1a00:0x2d00]
Prints the stall-reason totals and the hottest instructions (samples, reasons).
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--kernel", default=None, help="substring of the kernel name (first match)")
a = ap.parse_args()
cmd = ["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
sel = next(k for k in range(len(starts) - 1) if a.kernel is None or a.kernel in rows[starts[k]][1])
print(rows[starts[sel]][1][:150])
rows = rows[starts[sel]:starts[sel + 1]]
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[i0]
body = [r for r in rows[i0 + 1:] if len(r) == len(hdr)]
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
S = hdr.index("Warp Stall Sampling (All Samples)")
X = hdr.index("Instructions Executed")
tot = {hdr[i]: 0 for i in st}
allS = 0
for r in body:
    allS += int(r[S] or 0)
    for i in st:
        tot[hdr[i]] += int(r[i] or 0)
print(f"samples {allS}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {k:28s} {v:9d} {100 * v / max(allS, 1):5.1f}%")
# instruction mix of executed instructions
mix = {}
for r in body:
    op = r[1].split()[0] if r[1].split() else "?"
    if op.startswith("@"):
        op = r[1].split()[1]
    op = op.split(".")[0]
    mix[op] = mix.get(op, 0) + int(r[X] or 0)
totx = sum(mix.values())
print("executed instruction mix:", ", ".join(f"{k} {100 * v / totx:.1f}%" for k, v in sorted(mix.items(), key=lambda kv: -kv[1])[:14]))
print("hottest instructions:")
body.sort(key=lambda r: -int(r[S] or 0))
for r in body[: a.top]:
    rs = sorted(((int(r[i] or 0), hdr[i][6:]) for i in st), reverse=True)[:3]
    print(f"  {r[0][-5:]} {int(r[S] or 0):7d} {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in rs if v))
