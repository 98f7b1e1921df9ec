#!/bin/bash
# Time every tools/tune_build/lib_*.so on the C2 bench (quick mode).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for so in tools/tune_build/lib_*.so; do
  tag=$(basename $so .so)
  for ct in f32; do
    DIFFOPT_LIB=$PWD/$so python bench.py --quick --no-cpu-baseline --steps 100 --compute $ct $TUNE_ARGS > gpurun_out/tune_${tag}_${ct}.json 2>gpurun_out/tune_${tag}_${ct}.err
    python -c "import json;d=json.load(open('gpurun_out/tune_${tag}_${ct}.json'));print('$tag $ct', d['value'], d['fwd_gbs'], d['roofline']['achieved'])"
  done
done
