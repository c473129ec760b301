#!/bin/bash
# BASELINE.json configs at 1 GPU (extra bench lines, not the headline):
# C1 water/STO-3G, C2 benzene/6-31G*, C3 (H2O)_16/cc-pVDZ, C4 (H2O)_64/cc-pVDZ,
# C5: idealised H-(Ala)_n-OH strands at cc-pVTZ (taxol coordinates are unavailable offline).
O=gpurun_out/${1:-configs}; mkdir -p $O
run() { tag=$1; shift; timeout 600 python bench.py --no-cpu --steps 5 --warmup 3 "$@" > $O/$tag.json 2> $O/$tag.err; \
  python -c "import json,sys; d=json.loads(open('$O/$tag.json').read().strip().splitlines()[-1]); print('$tag', d['config']['n_basis'], d['quartets_per_build'], round(d['ms_per_step'],3), '%.3e'%d['value'], round(d['roofline']['build_frac'],3) if d.get('roofline') else None)"; }
run c1_water_sto3g --geom water --basis sto-3g --tau 0 --kappa 0
run c2_benzene_631gs --geom benzene --basis 6-31g* --tau 1e-10
run c3_w16_ccpvdz --waters 16 --basis cc-pvdz
run c4_w64_ccpvdz --waters 64 --basis cc-pvdz
run c4_w64_ccpvdz_tau12 --waters 64 --basis cc-pvdz --tau 1e-12
run c5_ala4_ccpvtz --geom ala4 --basis cc-pvtz
run c5_ala8_ccpvtz --geom ala8 --basis cc-pvtz
