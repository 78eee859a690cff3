#!/bin/bash
# c3: ncu of one band and one sparse attention launch inside the relay step
OUT=gpurun_out/c3attn; mkdir -p $OUT
NV="--nvtx --nvtx-include relay_step/"
LEAN="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --lean"
timeout 900 ncu $NV --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $LEAN > $OUT/l.log 2>&1
for spec in "attn_kernel:2" "attn_kernel:4"; do
  pat=${spec%%:*}; skip=${spec##*:}
  timeout 600 ncu $NV --set full --import-source on --clock-control none -k regex:$pat -s $skip -c 1 -o $OUT/full_${pat}_$skip $LEAN > $OUT/ncu_$skip.log 2>&1
done
echo done
