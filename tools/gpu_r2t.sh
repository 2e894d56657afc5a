# round 2 (t): first tcgen05 filter run: small parity tests under a timeout, then C4 A/B
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "dense_tiles or config1 or cluster or edge" 2>&1 | tail -15 > gpurun_out/r2t_tests.txt
cat gpurun_out/r2t_tests.txt
for lib in m tc0; do for cfg in "4" "4 --mode nearest"; do
  echo "$lib | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 120 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r2t.txt
done; done
cat gpurun_out/r2t.txt
