cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02ac; mkdir -p $OUT
for cfg in "X=0" "RK_ATTN_SPLITWAVES=100" "RK_ATTN_SPLITWAVES=100,RK_ATTN_SPLITDIV=1" "RK_ATTN_SPLITWAVES=100,RK_ATTN_MINPART=8"; do
  echo "== $cfg" >> $OUT/mb.txt
  env $(echo $cfg | tr ',' ' ') timeout 120 python tools/microbench.py rows >> $OUT/mb.txt 2>&1
done
