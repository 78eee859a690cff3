cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02q; mkdir -p $OUT
for cfg in "X=0" "RK_ATTN_MERGE=0" "RK_ATTN_DBG=1" "RK_ATTN_DBG=2" "RK_ATTN_DBG=3"; do
  echo "== $cfg" >> $OUT/mb.txt
  env $(echo $cfg | tr ',' ' ') timeout 120 python tools/microbench.py rows >> $OUT/mb.txt 2>&1
done
