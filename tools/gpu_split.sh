#!/bin/bash
for w in 1 2 4 1 2 4; do
  r=$(RK_ATTN_SPLITWAVES=$w timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --lean 2>/dev/null)
  echo "waves=$w c2 $r"
done
for w in 1 2 4; do
  r=$(RK_ATTN_SPLITWAVES=$w timeout 900 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu --lean 2>/dev/null)
  echo "waves=$w c3 $r"
done
