cd $GRAFT_REPO_ROOT
bash tools/r2_var.sh ws dirichlet
BRNG_LIB=tools/variants/ws.so timeout 900 python -m pytest tests/test_gpu_gamma.py tests/test_gpu_graphs.py tests/test_gpu_lda.py -x -q > gpurun_out/r2_ws_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_ws_tests.log
