cd $GRAFT_REPO_ROOT
timeout 1500 python tools/parity_audit.py > gpurun_out/r2_parity_audit.json 2> gpurun_out/r2_parity_audit.err; echo rc=$? >> gpurun_out/r2_parity_audit.err
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_all.log 2>&1; echo rc=$? >> gpurun_out/r2_gpu_all.log
