# round 2 (4o): final check of the committed build: GPU suite, default bench, wide fuzz campaign
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r4o_smoke.txt 2>&1
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r4o_tests.txt
python bench.py > gpurun_out/r4o_bench.json 2> gpurun_out/r4o_bench.err
for seed in 51 52 53 54 55 56; do
  SPIN_FUZZ_SEED=$seed SPIN_FUZZ_CASES=500 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k test_fuzz_against_oracle 2>&1 | tail -1 | sed "s/^/seed $seed x 500: /" >> gpurun_out/r4o_fuzz.txt
done
tail -2 gpurun_out/r4o_smoke.txt; cat gpurun_out/r4o_tests.txt gpurun_out/r4o_fuzz.txt; tail -c 400 gpurun_out/r4o_bench.json
