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
  # c2 step order: gemm_bf16_kernel #5 = band gate/up (layer 1), #11-#14 = first
  # sparse layer's QKV / W_o / gate/up / W_down; attn_kernel #0 prefix+suffix
  # layer, #1 band, #3 sparse; gemm_swap_kernel #0 = prefix+suffix gate/up
  for spec in "gemm_bf16_kernel:5:1" "gemm_bf16_kernel:11:4" "attn_kernel:0:1" "attn_kernel:1:1" "attn_kernel:3:1" \
              "gemm_swap_kernel:0:1" "realign_graft:0:1" "score_dh_kernel:0:1" "select_relay_kernel:0:1"; do
    pat=${spec%%:*}; rest=${spec#*:}; skip=${rest%%:*}; cnt=${rest##*:}
    timeout 900 ncu $NV --set full --import-source on --clock-control none -k regex:$pat -s $skip -c $cnt \
      -o $OUT/full_${pat}_$skip $LEAN > $OUT/ncu_${pat}_$skip.log 2>&1
  done
fi
echo done > $OUT/DONE
