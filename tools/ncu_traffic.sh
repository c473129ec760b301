#!/bin/bash
# DRAM traffic of the dominant class launch for bench.py's roofline.traffic:
# every kernel of class CLS (default 1000, (ps|ss)) in one tuned (H2O)_80 build,
# dram__bytes_read/write summed over the class's launches -> profiles/ncu_traffic.json
CLS=${1:-1000}
VAR=${2:-}   # kernel variant to measure (default: whatever --tune picks)
SET=""; [ -n "$VAR" ] && SET="--set $CLS=$VAR"
O=gpurun_out/traffic_$CLS; mkdir -p $O
timeout 1200 ncu --profile-from-start off --clock-control none --kernel-name-base demangled -k "regex:Cls$CLS," \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/traffic.csv \
  python tools/profile_build.py --waters 80 --builds 1 --tune $SET --profile-range --variants-json $O/variants.json > $O/log.txt 2>&1
python - "$O" "$CLS" <<'PY'
import csv, json, sys
O, cls = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(f"{O}/traffic.csv")) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
ui = hdr.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
per = {}
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    except ValueError:
        continue
    per.setdefault((r[ii], r[ki]), {})[r[mi]] = v
# the tuned build is the last one: keep the launches after the tune's (ids in order)
launches = sorted(per.items(), key=lambda kv: int(kv[0][0]))
var = json.load(open(f"{O}/variants.json")).get(cls, "?")
rd = sum(v.get("dram__bytes_read.sum", 0) for _, v in launches)
wr = sum(v.get("dram__bytes_write.sum", 0) for _, v in launches)
ms = sum(v.get("gpu__time_duration.sum", 0) for _, v in launches)
out = [{"workload": "(H2O)_80/cc-pvdz RHF Fock build (ERI + J/K), Schwarz tau=1e-10, kappa screen 1e-14",
        "cls": cls, "variant": var, "launches": len(launches),
        "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
        "kernel_ms_serialised": ms,
        "source": f"{O}/traffic.csv: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (tools/ncu_traffic.sh), "
                  f"variant {var}, summed over the class's {len(launches)} kernel launches"}]
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
PY
