# round 2 (3d): PASS1 for 768-thread CTAs only; configs + GPU tests
for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6"; do
  echo "m | $(SPIN_LIB_PATH=abbuild/m/libspin.so timeout 120 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r3d.txt
done
python -m pytest tests -m gpu -q 2>&1 | tail -4 >> gpurun_out/r3d.txt
cat gpurun_out/r3d.txt
