cd $GRAFT_REPO_ROOT
python tools/variant_time.py dirichlet > gpurun_out/r2_var_dir_raw.txt 2>&1
python tools/variant_time.py gamma > gpurun_out/r2_var_gamma_raw.txt 2>&1
timeout 900 python tools/lda_bench.py 10 > gpurun_out/r2_lda2.json 2> gpurun_out/r2_lda2.err; echo rc=$? >> gpurun_out/r2_lda2.err
