# round 2 (i): 512-thread G = 32 with dense tiles: dense_min sweep, stage breakdown, NEAREST; hetero test
python -m pytest tests/test_gpu_parity.py -x -q -k heterogeneous 2>&1 | grep -v "^$" | tail -30 > gpurun_out/r2i_tests.txt
run() { echo "$1 | $(env $1 SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py $2 2>&1 | tail -1)" >> gpurun_out/r2i.txt; }
for dm in 4 8 16 24; do run "SPIN_DENSE_MIN=$dm SPIN_DEBUG_G=32 SPIN_DEBUG_NT=512" "--config 4"; done
for sk in 1 2; do run "SPIN_DENSE_MIN=8 SPIN_DEBUG_SKIP=$sk SPIN_DEBUG_G=32 SPIN_DEBUG_NT=512" "--config 4"; done
for dm in 0 8 16; do run "SPIN_DENSE_MIN=$dm SPIN_DEBUG_G=32 SPIN_DEBUG_NT=512" "--config 4 --mode nearest"; done
for dm in 8 16; do run "SPIN_DENSE_MIN=$dm SPIN_DEBUG_G=32" "--config 2"; run "SPIN_DENSE_MIN=$dm SPIN_DEBUG_G=32" "--config 2 --mode nearest"; run "SPIN_DENSE_MIN=$dm SPIN_DEBUG_G=32" "--config 6"; done
cat gpurun_out/r2i_tests.txt gpurun_out/r2i.txt
