#!/bin/bash
OUT=gpurun_out/spin; mkdir -p $OUT
for d in 0 16 0 16; do
  echo "== dbg=$d"; RK_GEMM_DBG=$d timeout 200 python tools/microbench.py gemm 2>&1
  RK_GEMM_DBG=$d timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --lean > $OUT/b.json 2> $OUT/b.err; cat $OUT/b.json
done
