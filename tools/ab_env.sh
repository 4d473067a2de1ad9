#!/bin/bash
# A/B of an environment setting on the same box: ROUNDS alternating bench runs with each value of
# $VAR given.   VAR=FSA_ZERO_FIRST bash tools/ab_env.sh 0 1
ROUNDS=${ROUNDS:-3}
ARGS=${ARGS:---no-cpu --no-alt --no-unfused --no-train --no-parity --steps 300}
for r in $(seq $ROUNDS); do
  for v in "$@"; do
    env $VAR=$v python bench.py $ARGS 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$VAR=$v', d['ms_per_step'], d['e2e']['value'], d['clocks'].get('samples'), d['clocks'].get('sm_mhz'), {k[2:]: round(v['ms']*1000, 1) for k, v in d.get('kernels', {}).items()})"
  done
done
