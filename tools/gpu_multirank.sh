#!/bin/bash
# Exercise bench.py's multi-rank path (sharding + all-reduce + max-over-ranks)
# with 2 ranks on one GPU over gloo (NCCL needs one GPU per rank).
O=gpurun_out/${1:-multirank}; mkdir -p $O
ERITILE_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --waters 16 --no-unscreened \
  > $O/bench2.json 2> $O/bench2.err
timeout 900 python bench.py --steps 3 --warmup 3 --waters 16 --no-unscreened --no-cpu > $O/bench1.json 2> $O/bench1.err
for f in bench1 bench2; do python -c "
import json; d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1])
print('$f', d['n_gpus'], d['quartets_per_build'], round(d['ms_per_step'],2), '%.3e'%d['value'], d['config']['parallelism'])"; done
tail -3 $O/bench2.err
