ROUNDS=2 ARGS="--no-cpu --no-alt --no-unfused --no-train --no-parity --steps 200" bash tools/ab.sh tools/ab/lib_w4.so tools/ab/lib_cpa.so
ROUNDS=1 ARGS="--config arxiv --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 200" bash tools/ab.sh tools/ab/lib_w4.so tools/ab/lib_cpa.so
FSA_LIB=tools/ab/lib_cpa.so python tools/timeline.py --reps 1 2>&1 | grep "hop1\|sample2\|multi"
