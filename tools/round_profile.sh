#!/bin/bash
# Everything the profiles/ directory records for one round: pytest -m gpu, smoke, the default
# bench line, the timeline trace, an ncu launch list of 3 eager steps and an ncu --set full capture
# of every kernel of one step, then the bench lines of the other BASELINE configs (with their CPU
# baselines) and the sampler's draw-loop peak.
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 300 python tools/timeline.py --reps 2 > gpurun_out/${TAG}_timeline.txt 2>&1
timeout 300 python tools/timeline.py --config reddit --reps 1 > gpurun_out/${TAG}_timeline_reddit.txt 2>&1
timeout 300 python tools/timeline.py --config arxiv --reps 1 > gpurun_out/${TAG}_timeline_arxiv.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python tools/profile_step.py --alpha 3.0 --steps 3 > /dev/null 2>&1
# one eager step = 4 forward + 8 backward launches (with the sparse re-zero); skip the first step
NK=${NK:-12}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ -s $NK -c $NK \
    -o gpurun_out/${TAG}_full -f python tools/profile_step.py --alpha 3.0 --steps 3 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_traffic.py gpurun_out/${TAG}_full.ncu-rep ${TAG} > gpurun_out/${TAG}_ncu_traffic.json 2>&1
timeout 900 python bench.py --config reddit --no-alt > gpurun_out/${TAG}_bench_reddit.json 2> gpurun_out/${TAG}_bench_reddit.err
timeout 900 python bench.py --config arxiv --no-alt > gpurun_out/${TAG}_bench_arxiv.json 2> gpurun_out/${TAG}_bench_arxiv.err
timeout 900 python bench.py --config products25 --no-alt > gpurun_out/${TAG}_bench_products25.json 2> gpurun_out/${TAG}_bench_products25.err
timeout 300 python tools/bench_draws.py --json gpurun_out/${TAG}_draw_peak.json > /dev/null 2>&1
ls gpurun_out | grep ${TAG}
