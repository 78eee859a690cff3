#!/bin/bash
# CTA-pair GEMM: kernel tests, then c2 bench with pairs off / auto.
OUT=gpurun_out/pair; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k gemm > $OUT/pytest_gemm.log 2>&1; echo "exit $?" >> $OUT/pytest_gemm.log
tail -2 $OUT/pytest_gemm.log
for pair in 0 1; do
  RK_GEMM_PAIR=$pair timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_pair$pair.json 2> $OUT/bench_pair$pair.err
  python -c "import json; d=json.load(open('$OUT/bench_pair$pair.json')); print('pair=$pair', d['ms_per_step'], d['value'], d['e2e']['value'])"
done
