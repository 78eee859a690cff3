#!/bin/bash
# GEMM: L2 prefetch of B x MM: microbench + c2 bench
OUT=gpurun_out/pf; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k gemm > $OUT/pytest_gemm.log 2>&1; echo "exit $?" >> $OUT/pytest_gemm.log
tail -2 $OUT/pytest_gemm.log
for cfg in "0 0" "8 0" "8 1" "16 1" "4 1"; do
  set -- $cfg
  echo "== prefetch=$1 mm=$2"
  RK_GEMM_PREFETCH=$1 RK_GEMM_MM=$2 timeout 200 python tools/microbench.py gemm 2>&1 | grep -v "^\[gemm"
  RK_GEMM_PREFETCH=$1 RK_GEMM_MM=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); print('bench', d['ms_per_step'], d['roofline']['frac'], d['kernels']['gemm_bf16_tcgen05']['ms'])"
done
