# round 2 (4v): wide fuzz campaign on the final build (10 seeds x 1000 cases)
for seed in 61 62 63 64 65 66 67 68 69 70; do
  SPIN_FUZZ_SEED=$seed SPIN_FUZZ_CASES=1000 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k test_fuzz_against_oracle 2>&1 | tail -1 | sed "s/^/seed $seed x 1000: /" >> gpurun_out/r4v_fuzz.txt
done
cat gpurun_out/r4v_fuzz.txt
