cd $GRAFT_REPO_ROOT
python tools/variant_time.py gamma > gpurun_out/r2_var_gamma.txt 2>&1
python tools/variant_time.py dirichlet > gpurun_out/r2_var_dir.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_gamma.py -x -q > gpurun_out/r2_t_gamma.log 2>&1
echo rc=$? >> gpurun_out/r2_t_gamma.log
