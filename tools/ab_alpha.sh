for i in 1 2; do
python bench.py --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 200 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('products', d['ms_per_step'], d['e2e']['value'])"
python bench.py --config reddit --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 100 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('reddit', d['ms_per_step'], d['e2e']['value'])"
python bench.py --config arxiv --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 200 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('arxiv', d['ms_per_step'], d['e2e']['value'])"
done
python tools/timeline.py --reps 1 2>&1 | cut -c1-100
