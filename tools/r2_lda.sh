cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_lda.py -x -q > gpurun_out/r2_lda_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_lda_tests.log
timeout 900 python tools/lda_bench.py 10 > gpurun_out/r2_lda.json 2> gpurun_out/r2_lda.err; echo rc=$? >> gpurun_out/r2_lda.err
