#!/bin/bash
OUT=gpurun_out/pf2; mkdir -p $OUT
for pf in 0 4 8 16 0; do
  RK_GEMM_PREFETCH=$pf timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --lean > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); print('pf=$pf', d['ms_per_step'])"
done
