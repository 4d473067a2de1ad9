for cfg in products reddit arxiv; do for m in 1 2; do
  FSA_HOP1=$m python bench.py --config $cfg --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 150 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$cfg', $m, d['ms_per_step'], d['e2e']['value'])"
done; done
