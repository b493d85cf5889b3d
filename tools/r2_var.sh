# usage: bash tools/r2_var.sh "<kernels>" "<variants>" [passes]  -- time build variants (tools/variants/*.so)
cd $GRAFT_REPO_ROOT
P=${3:-2}
for k in $1; do
  for r in $(seq $P); do
    python tools/variant_time.py $k $(for v in $2; do echo tools/variants/$v.so; done)
  done
done > gpurun_out/var.txt 2>&1
