# round 2 (f): dense lane-per-centre tiles on the Morton-ordered cloud: GPU tests, then the
# dense_min sweep (measurement build) on C4 / C2 (BILINEAR and NEAREST)
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2f_tests.txt
for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6"; do
  for dm in 0 4 8 12 16; do
    SPIN_DENSE_MIN=$dm SPIN_LIB_PATH=abbuild/m/libspin.so timeout 300 python bench.py --config $cfg --steps 3 --no-cpu-baseline --no-e2e --no-dls > /tmp/o.json 2>/dev/null
    python -c "
import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('cfg $cfg dense_min $dm', round(d['roofline']['kernel_ms'],2), d['config']['G'], d['pairs']['candidate'], d['pairs']['accepted'], d['pairs']['fp64_fallbacks'])" >> gpurun_out/r2f_sweep.txt 2>&1
  done
done
cat gpurun_out/r2f_tests.txt gpurun_out/r2f_sweep.txt
