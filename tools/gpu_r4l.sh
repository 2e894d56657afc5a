# round 2 (4l): seeded fuzz campaign against the oracle on the final round-2 build (3 seeds x 300 cases)
for seed in 41 42 43; do
  SPIN_FUZZ_SEED=$seed SPIN_FUZZ_CASES=300 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -k test_fuzz_against_oracle 2>&1 | tail -2 | sed "s/^/seed $seed: /" >> gpurun_out/r4l_fuzz.txt
done
cat gpurun_out/r4l_fuzz.txt
