# usage: bash tools/r2_ncu_lda.sh -- source-level capture of the LDA consumer (INLINE, bench shape)
cd $GRAFT_REPO_ROOT
python tools/run_lda.py 0 > gpurun_out/r2_lda_run.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -s 1 -c 1 -k regex:lda_consumer \
  -o gpurun_out/r2_src_lda_new python tools/run_lda.py 0 64 150 1 > gpurun_out/r2_src_lda_new.log 2>&1
