#!/bin/bash
# Time every tools/tune_build/lib_*.so on the C2 bench (quick mode), in
# ROUNDS alternating passes so box drift hits every variant alike.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for r in $(seq 1 ${ROUNDS:-2}); do
for so in tools/tune_build/lib_*.so; do
  tag=$(basename $so .so)
  DIFFOPT_LIB=$PWD/$so python bench.py --quick --no-cpu-baseline --no-maml --no-secondary --steps 200 $TUNE_ARGS > gpurun_out/tune_${tag}.json 2>gpurun_out/tune_${tag}.err
  python -c "import json;d=json.load(open('gpurun_out/tune_${tag}.json'));print('r$r $tag', d['value'], d['fwd_gbs'], d['roofline']['achieved'], d['roofline']['frac'])"
done
done
