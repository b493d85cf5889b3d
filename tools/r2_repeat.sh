cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_rep$i.json 2> gpurun_out/r2_rep$i.err
done
