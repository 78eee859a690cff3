#!/bin/bash
OUT=gpurun_out/cfg5; mkdir -p $OUT
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_c2.json 2> $OUT/bench_c2.err
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
for c in c2 c3 c4; do
  python -c "import json; d=json.load(open('$OUT/bench_$c.json')); r=d['roofline']; print('$c', d['ms_per_step'], r['achieved'], r['frac'], r['launches_per_step'], r['gemm_ms_per_step'], d['kernels'].get('attention_bf16_tcgen05'), d['kernels'].get('gemv_bf16'))"
done
