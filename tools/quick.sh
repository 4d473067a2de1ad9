#!/bin/bash
# GPU tests + products / reddit bench (+ optional timeline) in one gpurun call; prints a summary.
rm -f gpurun_out/bp.json gpurun_out/br.json gpurun_out/bp.err gpurun_out/br.err gpurun_out/pytest_gpu.log gpurun_out/tl_p.txt
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1500 -- 'timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log; python bench.py --no-cpu --no-alt --steps 200 > gpurun_out/bp.json 2>gpurun_out/bp.err; python bench.py --config reddit --no-cpu --no-alt --steps 50 > gpurun_out/br.json 2> gpurun_out/br.err; '"${TL:+python tools/timeline.py --reps 1 > gpurun_out/tl_p.txt 2>&1; }$EXTRA" 2>&1 | tail -1
tail -2 gpurun_out/pytest_gpu.log
for f in bp br; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d['ms_per_step'],d['e2e']['value'], {k[2:]:round(v['ms']*1000,1) for k,v in d['kernels'].items()})"; done
[ -f gpurun_out/tl_p.txt ] && cut -c1-100 gpurun_out/tl_p.txt
