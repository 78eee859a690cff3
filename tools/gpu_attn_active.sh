#!/bin/bash
OUT=gpurun_out/aa; mkdir -p $OUT
NV="--nvtx --nvtx-include relay_step/"
for cfg in c2 c3; do
  LEAN="python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu --lean"
  for skip in 1 4; do
    timeout 600 ncu $NV --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:attn_kernel -s $skip -c 1 --csv $LEAN 2>/dev/null | grep -E "gpu__time|cycles_active|cycles_elapsed|tensor" | awk -F'","' -v c=$cfg -v s=$skip '{print c, s, $(NF-2), $NF}'
  done
done
