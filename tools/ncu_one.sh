#!/bin/bash
# ncu --set full of one kernel (regex $K) in step 2 of profile_step.py
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${K} -s ${SKIP:-1} -c ${COUNT:-1} \
  -o gpurun_out/${TAG:-one} -f python tools/profile_step.py --alpha ${ALPHA:-3.0} --steps 3 ${PS_ARGS} > gpurun_out/ncu_${TAG:-one}.log 2>&1
tail -2 gpurun_out/ncu_${TAG:-one}.log
