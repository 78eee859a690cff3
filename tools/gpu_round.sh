#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (both arms), ncu launch list and
# full captures of the hot kernels. Usage (from the repo root, on the box):
#   bash tools/gpu_round.sh <tag> [parts]
# parts: any of test,smoke,bench,ref,launches,ncu (default: all)
TAG=${1:-run}
PARTS=${2:-test,smoke,bench,ref,launches,ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
has() { [[ ",$PARTS," == *",$1,"* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> $OUT/gpu.txt
if has test; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
fi
if has bench; then
  timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
fi
if has ref; then
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --lean > $OUT/launches_bench.log 2>&1
fi
if has ncu; then
  for pat in gemm_bf16_kernel attn_kernel realign_graft_kernel score_kernel select_relay_kernel; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$pat -s 40 -c 2 \
      -o $OUT/full_$pat python bench.py --steps 1 --warmup 3 --no-cpu --lean > $OUT/ncu_$pat.log 2>&1
  done
fi
echo done > $OUT/DONE
