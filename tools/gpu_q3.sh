#!/bin/bash
OUT=gpurun_out/q3; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bf16.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > $OUT/p.log 2>&1; tail -1 $OUT/p.log
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --lean 2>/dev/null; done
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --lean 2>/dev/null
