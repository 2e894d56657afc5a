# round 2 (n): two live rows per dense step, parallel AND chains in the filter pre-pass
python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r2n_tests.txt
for lib in m dr1; do for cfg in "4" "4 --mode nearest" "2" "6"; do
  echo "$lib | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r2n.txt
done; done
for sk in 1 2; do echo "m skip $sk | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py --config 4 2>&1 | tail -1)" >> gpurun_out/r2n.txt; done
cat gpurun_out/r2n_tests.txt gpurun_out/r2n.txt
