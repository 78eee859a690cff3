#!/bin/bash
OUT=gpurun_out/cfg3; mkdir -p $OUT
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "import json; d=json.load(open('$OUT/bench_$c.json')); print('$c', d['ms_per_step'], d['value'], d['ttft_ms'], d['full_prefill_ttft_ms'], d['roofline']['achieved'], d['e2e']['ttft_ms'], d['kernels']['attention_bf16_tcgen05'])"
done
