#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (both arms), an ncu launch list of
# exactly one relay step (NVTX range "relay_step" in bench.py) and --set full
# captures of the hot kernels inside that step. Usage (on the box):
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
  timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
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
NV="--nvtx --nvtx-include relay_step/"
LEAN="python bench.py --steps 1 --warmup 0 --no-cpu --lean"
if has launches; then
  timeout 900 ncu $NV --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    $LEAN > $OUT/launches_bench.log 2>&1
fi
if has ncu; then
  # kernel regex : launches to skip inside the step (c2: attention launch 1 = band layer 1,
  # launch 3 = first sparse layer; GEMM launch 6 = band gate/up)
  for spec in "gemm_bf16_kernel:6" "attn_kernel:1" "attn_kernel:3" "realign_graft:0" "score_dh_kernel:0" \
              "select_relay_kernel:0"; do
    pat=${spec%%:*}; skip=${spec##*:}
    timeout 600 ncu $NV --set full --import-source on --clock-control none -k regex:$pat -s $skip -c 1 \
      -o $OUT/full_${pat}_$skip $LEAN > $OUT/ncu_${pat}_$skip.log 2>&1
  done
fi
echo done > $OUT/DONE
