cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02ao; mkdir -p $OUT
for cfg in "X=0" "RK_ATTN_SPLITDIV=3" "RK_ATTN_SPLITDIV=4,RK_ATTN_MINPART=2" "RK_ATTN_SPLITDIV=6,RK_ATTN_MINPART=2" "RK_ATTN_SPLITDIV=1.5"; do
  echo "== $cfg" >> $OUT/mb.txt
  env $(echo $cfg | tr ',' ' ') timeout 120 python tools/microbench.py rows >> $OUT/mb.txt 2>&1
done
