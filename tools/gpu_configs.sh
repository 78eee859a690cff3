#!/bin/bash
# c3 / c4 bench lines with the current kernels
OUT=gpurun_out/cfg; mkdir -p $OUT
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "import json; d=json.load(open('$OUT/bench_$c.json')); print('$c', d['ms_per_step'], d['value'], d['unit'], d['roofline']['achieved'], d['roofline']['frac'], d.get('full_prefill_ms'), d['e2e']['ttft_ms'])"
done
