# round 2 (y): C2 stage breakdown and the NO_SORT / NO_DENSE controls
run() { echo "$1 | $(env $1 SPIN_LIB_PATH=abbuild/m/libspin.so timeout 120 python tools/one_call.py $2 2>&1 | tail -1)" >> gpurun_out/r2y.txt; }
for m in bilinear nearest; do
  for sk in 0 1 2; do run "SPIN_DEBUG_SKIP=$sk" "--config 2 --mode $m"; done
  run "X=1" "--config 2 --mode $m --flags 0x4"
  run "X=1" "--config 2 --mode $m --flags 0x80"
  run "SPIN_DENSE_MIN=4" "--config 2 --mode $m"
  run "SPIN_DENSE_MIN=16" "--config 2 --mode $m"
  run "SPIN_DEBUG_G=32" "--config 2 --mode $m"
  run "SPIN_DEBUG_G=32 SPIN_DEBUG_NT=512" "--config 2 --mode $m"
done
cat gpurun_out/r2y.txt
