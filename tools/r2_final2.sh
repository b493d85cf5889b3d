# End-of-round bundle on the final code: GPU tests, smoke, the bench line,
# the ncu launch list + --set full captures, the LDA measurement.
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f2_build.log 2>&1
bash tools/r2_final.sh
bash tools/r2_prof.sh
python tools/lda_bench.py 10 > gpurun_out/f2_lda.json 2> gpurun_out/f2_lda.err
echo done
