#!/bin/bash
for cfg in "4 2" "2 2" "2 4" "3 3" "4 2" "2 8"; do
  set -- $cfg
  r=$(RK_ATTN_MINPART=$1 RK_ATTN_SPLITDIV=$2 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --lean 2>/dev/null)
  echo "minpart=$1 div=$2 $r"
done
