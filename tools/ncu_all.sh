#!/bin/bash
# ncu --set full of every kernel of one steady-state fused 2-hop step (step 2 of 3).
mkdir -p gpurun_out
ALPHA=${ALPHA:-3.0}
TAG=${TAG:-all}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ -s ${SKIP:-10} -c ${COUNT:-10} \
  -o gpurun_out/${TAG} -f python tools/profile_step.py --alpha $ALPHA --steps 3 > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log
