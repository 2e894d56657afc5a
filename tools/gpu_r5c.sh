# round 2 (5c): two live rows per dense-walk step for NEAREST on the 512-thread launch: GPU suite, timings, bench
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/r5c_check.txt
for cfg in "4" "4 --mode nearest" "2" "2 --mode nearest" "6"; do
  echo "cfg $cfg | $(timeout 300 python tools/one_call.py --config $cfg 2>&1 | tail -1 | cut -c1-75)" >> gpurun_out/r5c_check.txt
done
python bench.py 2> gpurun_out/r5c_bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])" >> gpurun_out/r5c_check.txt
SPIN_FUZZ_SEED=71 SPIN_FUZZ_CASES=1000 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k test_fuzz_against_oracle 2>&1 | tail -1 | sed "s/^/fuzz seed 71 x 1000: /" >> gpurun_out/r5c_check.txt
cat gpurun_out/r5c_check.txt
