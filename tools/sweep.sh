#!/bin/bash
# bench lines for every BASELINE.json config (device-resident + e2e + CPU oracle baseline)
mkdir -p gpurun_out/sweep
for cfg in products reddit arxiv products25; do
  for a in 3.0 2.1; do
    timeout 900 python bench.py --config $cfg --alpha $a --no-alt --steps ${STEPS:-100} --cpu-seconds 5 \
      > gpurun_out/sweep/${cfg}_a${a}.json 2> gpurun_out/sweep/${cfg}_a${a}.err
    echo "$cfg $a rc=$?"
  done
done
