cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_gibbs.py tests/test_gpu_shard_2proc.py -x -q > gpurun_out/r2_b1_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_b1_tests.log
timeout 600 python bench.py --small --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2_b1_small.json 2> gpurun_out/r2_b1_small.err; echo rc=$? >> gpurun_out/r2_b1_small.err
BRNG_BENCH_DEVICE=0 BRNG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/r2_b1_n2gloo.json 2> gpurun_out/r2_b1_n2gloo.err; echo rc=$? >> gpurun_out/r2_b1_n2gloo.err
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_b1_bench.json 2> gpurun_out/r2_b1_bench.err; echo rc=$? >> gpurun_out/r2_b1_bench.err
