cd $GRAFT_REPO_ROOT
BRNG_BENCH_DEVICE=0 BRNG_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_n2e2e.json 2> gpurun_out/r2_n2e2e.err; echo rc=$? >> gpurun_out/r2_n2e2e.err
/usr/bin/time -v timeout 1200 python bench.py > gpurun_out/r2_default.json 2> gpurun_out/r2_default.err; echo rc=$? >> gpurun_out/r2_default.err
timeout 900 python bench.py --scaling weak --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_weak1.json 2> gpurun_out/r2_weak1.err; echo rc=$? >> gpurun_out/r2_weak1.err
/usr/bin/time -v timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo rc=$? >> gpurun_out/r2_ref.err
