cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02ck; mkdir -p $OUT
for i in 1 2; do for mp in 4 6; do
  RK_ATTN_MINPART=$mp timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/c2_mp${mp}_$i.json 2>/dev/null
done; done
for mp in 4 6; do RK_ATTN_MINPART=$mp timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > $OUT/c4_mp${mp}.json 2>/dev/null; done
