# usage: bash tools/r2_ncu_src.sh   -- source-level --set full captures of the
# current Gamma (cfg3) and Dirichlet (cfg4) kernels (gpurun_out/r2_src_*.ncu-rep)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_src_build.log 2>&1
for k in gamma:gamma_kernel dirichlet:dirichlet_smem; do
  n=${k%%:*}; re=${k##*:}
  timeout 600 ncu --set full --import-source on --clock-control none -s 1 -c 1 -k regex:"$re" \
    -o gpurun_out/r2_src4_$n python tools/run_kernel.py $n > gpurun_out/r2_src4_$n.log 2>&1
done
