#!/bin/bash
# c3 / c4 bench lines and the c5 sweep with the current kernels
OUT=gpurun_out/cfg2; mkdir -p $OUT
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "import json; d=json.load(open('$OUT/bench_$c.json')); print('$c', d['ms_per_step'], d['value'], d['ttft_ms'], d['full_prefill_ttft_ms'], d['roofline']['achieved'], d['e2e']['ttft_ms'])"
done
timeout 2400 python tools/sweep.py > $OUT/sweep_c5.jsonl 2> $OUT/sweep.err
tail -3 $OUT/sweep_c5.jsonl
