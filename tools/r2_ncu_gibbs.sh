# usage: bash tools/r2_ncu_gibbs.sh TAG -- source-level --set full capture of the cfg5 Gibbs kernel
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_gb_build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -c 1 -k regex:'gibbs_kernel' \
  -o gpurun_out/r2_src_gibbs_$1 python tools/run_kernel.py gibbs > gpurun_out/r2_src_gibbs_$1.log 2>&1
