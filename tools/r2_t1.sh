cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -k "gibbs or graphs or abi_errors or batch_fill or gamma or dirichlet" > gpurun_out/r2_t1.log 2>&1
echo rc=$? >> gpurun_out/r2_t1.log
