cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ./oracle/_ref/engine_tests_on_dropin > gpurun_out/r02b_engine_tests_on_dropin.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_engine_tests_on_dropin.log
timeout 1800 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r02b_pytest_gpu.log 2>&1
cp gpurun_out/bf16_error_*.json gpurun_out/ 2>/dev/null
