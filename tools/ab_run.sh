ROUNDS=2 ARGS="--no-cpu --no-alt --no-unfused --no-train --no-parity --steps 200" bash tools/ab.sh tools/ab/lib_cur.so tools/ab/lib_r4.so
ROUNDS=1 ARGS="--config reddit --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 100" bash tools/ab.sh tools/ab/lib_cur.so tools/ab/lib_r4.so
ROUNDS=1 ARGS="--alpha 2.1 --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 30" bash tools/ab.sh tools/ab/lib_cur.so tools/ab/lib_r4.so
