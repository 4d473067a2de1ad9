A="--config reddit --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 100"
run() { env "$@" python bench.py $A 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$*', d['ms_per_step'])"; }
run FSA_X=0
for v in 2 3 6 8; do run FSA_MULTI_CTAS=$v; done
run FSA_SEG_DIV=1
run FSA_HOP1=1
run FSA_COUNT_CTAS=16
run FSA_X=0
