#!/bin/bash
# compute-sanitizer gate: memcheck, racecheck (shared-memory hazards), synccheck
# and initcheck over smoke(), the small golden parity cases and the training step's head / AdamW kernels.  Logs: gpurun_out/${TAG}_sanitize_*.log
mkdir -p gpurun_out
TAG=${TAG:-r02}
CS="compute-sanitizer --print-limit 50 --error-exitcode 99"
SMOKE="python -c 'import __graft_entry__ as g; g.smoke()'"
GOLD="python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k 'golden_cases or config1 or hub or wide or half or padded or sparse'"
# the first hop's piece queue (hub roots: pieces queued across warps, tagged items, global winners)
QUEUE="python -m pytest tests/test_gpu_large.py -m gpu -q -x -k 'piece_queue'"
# the training step's head row kernel and AdamW kernels (cp.async ring, last-CTA step count)
HEAD="python -m pytest tests/test_gpu_train.py -m gpu -q -x -k 'sage_head or adamw_kernel'"
for tool in memcheck racecheck synccheck initcheck; do
  log=gpurun_out/${TAG}_sanitize_${tool}.log
  : > $log
  cmds=("$SMOKE" "$GOLD" "$HEAD")
  if [ "$tool" = memcheck ] || [ "$tool" = racecheck ]; then cmds+=("$QUEUE"); fi
  for cmd in "${cmds[@]}"; do
    echo "### $tool: $cmd" >> $log
    eval timeout 1500 $CS --tool $tool $cmd >> $log 2>&1
    echo "### exit=$?" >> $log
  done
done
grep -H "ERROR SUMMARY\|### exit" gpurun_out/${TAG}_sanitize_*.log
