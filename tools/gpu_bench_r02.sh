# Round-2 measurement bundle (run under gpurun from the repo root): every
# profiles/r02_* file is produced by one of these steps.
set -x
# GPU tests, smoke, the bench line (20 steps), ncu launch list of one step
bash tools/r2_final.sh
# --set full captures of every hot kernel (+ the 2^21-chain cfg5 shard) and the LDA launch list
bash tools/r2_prof.sh
# full-size parity audit (every sample against the oracle, relaxations counted)
python tools/parity_audit.py > gpurun_out/r2_parity_audit.json 2> gpurun_out/r2_parity_audit.err
# the LDA consumer (N4): three deviate sources, two shapes
python tools/lda_bench.py 10 > gpurun_out/r2_lda.json 2> gpurun_out/r2_lda.err
# the reference arm and the N = 2 plumbing on one GPU
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err
BRNG_BENCH_DEVICE=0 BRNG_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 \
  --warmup 3 --no-cpu-baseline > gpurun_out/r2_n2e2e.json 2> gpurun_out/r2_n2e2e.err
# summaries: python tools/ncu_summary.py profiles/r02_ncu gpurun_out/rf_launches.csv gpurun_out/*.ncu-rep
echo done
