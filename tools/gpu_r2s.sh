# round 2 (s): restored K/w operands, tensor-core rule at 25%; configs + GPU tests
for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6"; do
  echo "m | $(SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r2s.txt
done
python tools/diag_dense.py > gpurun_out/r2s_diag.txt 2>&1
python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/r2s_tests.txt
cat gpurun_out/r2s_tests.txt gpurun_out/r2s.txt gpurun_out/r2s_diag.txt
