cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02o; mkdir -p $OUT
for cfg in "X=0" "RK_ATTN_MERGE=0" "RK_ATTN_PACK=0" "RK_ATTN_PACK=0,RK_ATTN_MERGE=0" "RK_PDL=0" "RK_PDL=0,RK_ATTN_MERGE=0" "RK_ATTN_SPLITWAVES=100" "RK_ATTN_SPLITWAVES=100,RK_ATTN_MERGE=0"; do
  echo "== $cfg" >> $OUT/mb.txt
  env $(echo $cfg | tr ',' ' ') timeout 120 python tools/microbench.py rows >> $OUT/mb.txt 2>&1
done
timeout 120 python tools/attn_trace.py 4032 4032 32 8 64 > $OUT/attn_trace_band.txt 2>&1
