# usage: bash tools/r2_ncu_var.sh <variant-name> <kernel: gamma|dirichlet|...> <regex>
cd $GRAFT_REPO_ROOT
BRNG_LIB=tools/variants/$1.so ncu --set full --import-source on --clock-control none -s 1 -c 1 -k regex:"$3" -o gpurun_out/r2_full_$2_$1 python tools/run_kernel.py $2 > gpurun_out/r2_ncu_$2_$1.log 2>&1
