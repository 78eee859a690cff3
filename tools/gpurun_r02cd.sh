cd $GRAFT_REPO_ROOT; OUT=gpurun_out/r02cd; mkdir -p $OUT
for sw in 1 2 3; do for mp in 2 3 4 6; do for sd in 1 2; do
  echo -n "SPLITWAVES=$sw MINPART=$mp SPLITDIV=$sd " >> $OUT/sweep.txt
  RK_ATTN_SPLITWAVES=$sw RK_ATTN_MINPART=$mp RK_ATTN_SPLITDIV=$sd timeout 120 python tools/microbench.py rows 2>&1 | tr '\n' ' ' >> $OUT/sweep.txt; echo >> $OUT/sweep.txt
done; done; done
