# Full verification + measurement bundle on the current code.
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/rf_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/rf_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; echo rc=$? >> gpurun_out/rf_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/rf_bench.json 2> gpurun_out/rf_bench.err; echo rc=$? >> gpurun_out/rf_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/rf_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/rf_ncu_list.log 2>&1
ncu --set full --import-source on --clock-control none -s 1 -c 1 -k regex:'dirichlet' -o gpurun_out/rf_full_dirichlet python tools/run_kernel.py dirichlet > gpurun_out/rf_ncu_dirichlet.log 2>&1
echo done
