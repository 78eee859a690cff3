#!/bin/bash
OUT=gpurun_out/attn2; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k attention > $OUT/p.log 2>&1; tail -1 $OUT/p.log
for pm in 0x88 0xAA 0x92 0; do
  echo "== poly $pm"
  RK_ATTN_POLY=$pm timeout 200 python tools/microbench.py attn 2>&1
done
for pm in 0x88 0xAA; do
  RK_ATTN_POLY=$pm timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); print('bench poly=$pm', d['ms_per_step'], d['kernels']['attention_bf16_tcgen05'])"
done
