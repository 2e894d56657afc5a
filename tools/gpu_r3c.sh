# round 2 (3c): pre-pass phase with prefetched fragment tiles (PASS1) A/B + GPU tests
for lib in m p0 p2; do for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6"; do
  echo "$lib | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 120 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r3c.txt
done; done
for sk in 1 2; do echo "m skip $sk | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/m/libspin.so timeout 120 python tools/one_call.py --config 4 2>&1 | tail -1)" >> gpurun_out/r3c.txt; done
python -m pytest tests -m gpu -q 2>&1 | tail -4 >> gpurun_out/r3c.txt
cat gpurun_out/r3c.txt
