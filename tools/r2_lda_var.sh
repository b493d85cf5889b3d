# usage: bash tools/r2_lda_var.sh "<variants>"  -- LDA bench per build variant
cd $GRAFT_REPO_ROOT
for v in $1; do echo "== $v"; BRNG_LIB=tools/variants/$v.so python tools/lda_bench.py 5 | python -c "
import json,sys; d=json.load(sys.stdin)
for s in ('headline','rng_heavy'): print(s, {m: d[s][m]['ms_per_iteration'] for m in ('inline','ring','bulk')})"; done > gpurun_out/lda_var.txt 2>&1
