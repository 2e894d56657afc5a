# round 2 (4h): default build after the accept-path trims: full GPU suite, timing per config
python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/r4h_tests.txt
for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6" "3" "5" "5 --W 24"; do
  echo "cfg $cfg | $(timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r4h_times.txt
done
cat gpurun_out/r4h_tests.txt gpurun_out/r4h_times.txt
