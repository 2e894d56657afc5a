# round 2 (u): tcgen05 filter with an opportunistic issuer, 3 A buffers, 4 TMEM tiles per warpgroup
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "dense_tiles or config1 or cluster or edge" 2>&1 | tail -15 > gpurun_out/r2u_tests.txt
cat gpurun_out/r2u_tests.txt
for lib in m tc0; do for cfg in "4" "4 --mode nearest"; do
  echo "$lib | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 120 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r2u.txt
done; done
for sk in 1 2; do echo "m skip $sk | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/m/libspin.so timeout 120 python tools/one_call.py --config 4 2>&1 | tail -1)" >> gpurun_out/r2u.txt; done
cat gpurun_out/r2u.txt
