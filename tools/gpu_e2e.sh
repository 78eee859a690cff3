#!/bin/bash
OUT=gpurun_out/e2e; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_parity.py -q -x -k "async or upload" > $OUT/p.log 2>&1; tail -1 $OUT/p.log
RK_XFER_SPLIT=1 timeout 300 python -m pytest tests/test_gpu_bf16.py tests/test_gpu_parity.py -q -x -k "async or upload" > $OUT/p2.log 2>&1; tail -1 $OUT/p2.log
for sp in 0 1 0 1; do
  RK_XFER_SPLIT=$sp timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); e=d['e2e']; print('split=$sp', d['ms_per_step'], e['ttft_ms'], e['upload_only_ms'], e['h2d_gbs'])"
done
