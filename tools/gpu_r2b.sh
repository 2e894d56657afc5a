set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster or widths or schedule_invariance or fuzz or carries" > gpurun_out/r2b_tests.log 2>&1; tail -3 gpurun_out/r2b_tests.log
for i in 1 2; do
timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-dls > gpurun_out/r2b_c4_cl.json 2>gpurun_out/r2b_c4_cl.err
SPIN_NO_CLUSTER=1 SPIN_LIB_PATH=abbuild/measure/libspin.so timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-dls > gpurun_out/r2b_c4_nocl.json 2>&1
SPIN_LIB_PATH=abbuild/measure/libspin.so timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-dls --mode nearest > gpurun_out/r2b_c4n_cl.json 2>&1
SPIN_NO_CLUSTER=1 SPIN_LIB_PATH=abbuild/measure/libspin.so timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e --no-dls --mode nearest > gpurun_out/r2b_c4n_nocl.json 2>&1
for f in r2b_c4_cl r2b_c4_nocl r2b_c4n_cl r2b_c4n_nocl; do python -c "
import json,sys; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2), d['config']['G'], d['pairs']['candidate'], d['clocks']['sm_mhz'])" ; done
done
