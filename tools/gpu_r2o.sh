# round 2 (o): single AND chain restored; two rows per dense step A/B; dense diag
python tools/diag_dense.py > gpurun_out/r2o_diag.txt 2>&1
for lib in m dr1; do for cfg in "4" "4 --mode nearest" "2" "6"; do
  echo "$lib | $(SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1)" >> gpurun_out/r2o.txt
done; done
for sk in 1 2; do echo "m skip $sk | $(SPIN_DEBUG_SKIP=$sk SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python tools/one_call.py --config 4 2>&1 | tail -1)" >> gpurun_out/r2o.txt; done
cat gpurun_out/r2o_diag.txt gpurun_out/r2o.txt
