# A/B of the two-CTA cluster variant knobs on C4 (measurement builds, abbuild/m*)
for lib in m0 m1 m2 m3; do
  for mode in bilinear nearest; do
    SPIN_LIB_PATH=abbuild/$lib/libspin.so timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-dls --mode $mode > gpurun_out/r2c_${lib}_${mode}.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/r2c_${lib}_${mode}.json').read().strip().splitlines()[-1]); print('$lib $mode', round(d['ms_per_step'],2), d['config']['G'], d['clocks']['sm_mhz'])"
  done
done
SPIN_NO_CLUSTER=1 SPIN_LIB_PATH=abbuild/m0/libspin.so timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-dls --mode nearest | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('m0 nocluster nearest', round(d['ms_per_step'],2), d['config']['G'])"
