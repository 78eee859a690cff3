cd $GRAFT_REPO_ROOT
bash tools/gpu_round.sh r02fin4
OUT=gpurun_out/r02fin4
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitizer_$tool.log 2>&1
  echo "exit $?" >> $OUT/sanitizer_$tool.log
done
