cd $GRAFT_REPO_ROOT
s=$(date +%s.%N); timeout 1200 python bench.py > gpurun_out/r2_default.json 2> gpurun_out/r2_default.err; echo rc=$? >> gpurun_out/r2_default.err; e=$(date +%s.%N); echo "wall $(echo "$e - $s" | bc)" >> gpurun_out/r2_default.err
s=$(date +%s.%N); timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo rc=$? >> gpurun_out/r2_ref.err; e=$(date +%s.%N); echo "wall $(echo "$e - $s" | bc)" >> gpurun_out/r2_ref.err
