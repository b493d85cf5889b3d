cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_lda.py -q -x > gpurun_out/lda_tests.log 2>&1
for v in lda_old lda_new; do echo $v; BRNG_LIB=tools/variants/$v.so python tools/lda_hash.py; done > gpurun_out/lda_hash.txt 2>&1
python tools/lda_bench.py > gpurun_out/lda_bench.json 2> gpurun_out/lda_bench.err
