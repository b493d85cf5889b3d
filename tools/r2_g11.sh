cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2_smoke.log
timeout 900 python -m pytest tests/test_gpu_lda.py -x -q > gpurun_out/r2_lda_tests2.log 2>&1; echo rc=$? >> gpurun_out/r2_lda_tests2.log
timeout 900 python tools/lda_bench.py 10 > gpurun_out/r2_lda3.json 2> gpurun_out/r2_lda3.err; echo rc=$? >> gpurun_out/r2_lda3.err
