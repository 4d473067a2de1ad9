#!/bin/bash
# A/B of library builds on the same box: ROUNDS alternating bench runs of each .so given
# (FSA_LIB), ms/step and e2e per run.   bash tools/ab.sh tools/ab/lib_base.so paper_2511_13645_b200/libfsa_b200.so
ROUNDS=${ROUNDS:-3}
ARGS=${ARGS:---no-cpu --no-alt --no-unfused --no-train --no-parity --steps 300}
for r in $(seq $ROUNDS); do
  for lib in "$@"; do
    FSA_LIB=$lib python bench.py $ARGS 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$lib', d['ms_per_step'], d['e2e']['value'])"
  done
done
