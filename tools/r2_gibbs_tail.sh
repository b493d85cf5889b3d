cd $GRAFT_REPO_ROOT
for nc in 16777216 8388608 4194304 2097152 150000; do
  echo "nc=$nc" >> gpurun_out/r2_gibbs_tail.txt
  GIBBS_NC=$nc python tools/variant_time.py gibbs >> gpurun_out/r2_gibbs_tail.txt 2>&1
done
