cd $GRAFT_REPO_ROOT
bash tools/r2_var.sh spec gamma dirichlet
BRNG_LIB=tools/variants/dspec.so timeout 900 python -m pytest tests/test_gpu_gamma.py -x -q > gpurun_out/r2_spec_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_spec_tests.log
