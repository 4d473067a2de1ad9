ROUNDS=1 ARGS="--config reddit --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 100" bash tools/ab.sh tools/ab/lib_w2.so tools/ab/lib_w3.so
ROUNDS=1 ARGS="--config reddit --dtype fp32 --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 100" bash tools/ab.sh tools/ab/lib_w2.so tools/ab/lib_w3.so
ROUNDS=1 ARGS="--no-cpu --no-alt --no-unfused --no-train --no-parity --steps 200" bash tools/ab.sh tools/ab/lib_w2.so tools/ab/lib_w3.so
ROUNDS=1 ARGS="--config products25 --no-cpu --no-alt --no-unfused --no-train --no-parity --steps 200" bash tools/ab.sh tools/ab/lib_w2.so tools/ab/lib_w3.so
