# Round-1 measurement bundle (run under gpurun from the repo root):
#   bench line, ncu launch list of one bench step, --set full capture of each
#   kernel, and the microbenchmarks behind DESIGN.md §7.
set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
echo "ncu list rc=$?"
for k in gamma dirichlet gaussian uniform gibbs1; do
  ncu --set full --import-source on --clock-control none -s 1 -c 1 -k regex:'gamma_kernel|dirichlet|fill_|gibbs_' -o gpurun_out/full_$k python tools/run_kernel.py $k > gpurun_out/ncu_$k.log 2>&1
done
ncu --set full --import-source on --clock-control none -c 1 -k regex:'gibbs_kernel' -o gpurun_out/full_gibbs python tools/run_kernel.py gibbs > gpurun_out/ncu_gibbs.log 2>&1
# microbenchmarks (single-process, seconds each)
for u in ubench ubench2 ulat ulat2; do
  nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/$u.cu -o /tmp/$u && /tmp/$u > gpurun_out/$u.txt
done
WARM=1 python tools/lat_probe.py 148 1024 4736 > gpurun_out/lat_probe.txt
python tools/parity_audit.py > gpurun_out/parity_audit.json 2> gpurun_out/parity_audit.err
echo done
