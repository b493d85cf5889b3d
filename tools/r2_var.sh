# usage: bash tools/r2_var.sh tag kernel1 [kernel2 ...]: time every tools/variants/*.so
cd $GRAFT_REPO_ROOT
tag=$1; shift
for k in "$@"; do python tools/variant_time.py $k > gpurun_out/r2_var_${k}_$tag.txt 2>&1; done
