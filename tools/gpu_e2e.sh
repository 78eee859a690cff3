#!/bin/bash
# host-side bf16 conversion in the async upload: bench e2e over worker counts
OUT=gpurun_out/e2e; mkdir -p $OUT
for cfg in "0 16" "1 4" "1 8" "1 12" "0 16"; do
  set -- $cfg
  RK_HOST_CONVERT=$1 RK_HOST_THREADS=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); e=d['e2e']; print('hc=$1 thr=$2', d['ms_per_step'], e['ttft_ms'], e['upload_only_ms'], e['h2d_gbs'])"
done
