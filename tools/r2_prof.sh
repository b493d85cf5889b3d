# Round-2 profiling bundle: ncu launch list of one bench step, --set full
# captures of the hot kernels, LDA bulk-mode launch list.
cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_list.log 2>&1
echo "list rc=$?"
for k in gamma dirichlet gaussian uniform gibbs1; do
  ncu --set full --import-source on --clock-control none -s 1 -c 1 -k regex:'gamma_kernel|dirichlet|fill_|gibbs_' -o gpurun_out/r2_full_$k python tools/run_kernel.py $k > gpurun_out/r2_ncu_$k.log 2>&1
done
ncu --set full --import-source on --clock-control none -c 1 -k regex:'gibbs_kernel' -o gpurun_out/r2_full_gibbs python tools/run_kernel.py gibbs > gpurun_out/r2_ncu_gibbs.log 2>&1
GIBBS_NC=2097152 ncu --set full --import-source on --clock-control none -c 1 -k regex:'gibbs_kernel' -o gpurun_out/r2_full_gibbs_shard8 python tools/run_kernel.py gibbs > gpurun_out/r2_ncu_gibbs8.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2_lda_launches.csv python tools/lda_bench.py 2 > gpurun_out/r2_lda_ncu.log 2>&1
echo done
