# round 2 (h): dense tiles without per-pair mask bits (decide's far test), shared-window atomics
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2h_tests.txt
run() { echo "$1 | $(env $1 SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py $2 2>&1 | tail -1)" >> gpurun_out/r2h.txt; }
for dm in 0 4 8 16; do run "SPIN_DENSE_MIN=$dm" "--config 4"; done
for dm in 0 8; do run "SPIN_DENSE_MIN=$dm SPIN_DEBUG_G=32 SPIN_DEBUG_NT=512" "--config 4"; done
for sk in 1 2; do run "SPIN_DENSE_MIN=8 SPIN_DEBUG_SKIP=$sk" "--config 4"; done
for dm in 0 4 8 16; do run "SPIN_DENSE_MIN=$dm" "--config 2"; run "SPIN_DENSE_MIN=$dm" "--config 2 --mode nearest"; done
for dm in 0 8; do run "SPIN_DENSE_MIN=$dm SPIN_NO_CLUSTER=1" "--config 4 --mode nearest"; run "SPIN_DENSE_MIN=$dm" "--config 6"; done
run "SPIN_DENSE_MIN=8" "--config 4 --mode nearest"
cat gpurun_out/r2h_tests.txt gpurun_out/r2h.txt
