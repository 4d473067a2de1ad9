# experiment knobs of the step (results never change): one bench run per setting, products
A="--no-cpu --no-alt --no-unfused --no-train --no-parity --steps 200"
run() { env "$@" python bench.py $A 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$*', d['ms_per_step'])"; }
run FSA_X=0
for v in 2 4; do run FSA_ZERO_CTAS=$v; done
for v in 4 16; do run FSA_COUNT_CTAS=$v; done
for v in 2 8; do run FSA_MULTI_CTAS=$v; done
run FSA_PLAN_PRIO=-1
run FSA_GATHER_PRIO=1
run FSA_X=0
