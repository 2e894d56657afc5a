# round 2 (q): bit-scan dense loop with two rows per step; A/B in one call + GPU tests
for lib in m dr1 d2; do for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6"; do
  echo "$lib | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r2q.txt
done; done
python tools/diag_dense.py > gpurun_out/r2q_diag.txt 2>&1
python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r2q_tests.txt
cat gpurun_out/r2q_tests.txt gpurun_out/r2q.txt
