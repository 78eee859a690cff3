#!/bin/bash
# GEMM bring-up: kernel tests, bf16 layer tests, then c2 bench with CSK off / on.
OUT=gpurun_out/csk; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x -k gemm > $OUT/pytest_gemm.log 2>&1; echo "exit $?" >> $OUT/pytest_gemm.log
tail -2 $OUT/pytest_gemm.log
timeout 400 python -m pytest tests/test_gpu_bf16.py -q -x > $OUT/pytest_bf16.log 2>&1; echo "exit $?" >> $OUT/pytest_bf16.log
tail -2 $OUT/pytest_bf16.log
RK_GEMM_CSK=0 timeout 200 python tools/microbench.py gemm > $OUT/mb_part.log 2>&1
timeout 200 python tools/microbench.py gemm > $OUT/mb_csk.log 2>&1
paste -d'\n' $OUT/mb_part.log $OUT/mb_csk.log
for csk in 0 1; do
  RK_GEMM_CSK=$csk timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $OUT/bench_csk$csk.json 2> $OUT/bench_csk$csk.err
  python -c "import json; d=json.load(open('$OUT/bench_csk$csk.json')); print('csk=$csk', d['ms_per_step'], d['value'], d['e2e']['value'])"
done
