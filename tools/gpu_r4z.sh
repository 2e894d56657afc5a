# round 2 (4z): one-off wide parity campaign on the final build (20,000 seeded images per config against
# the C++ oracle), logged like the default at-scale checks
SPIN_WIDE=1 SPIN_PARITY_LOG=gpurun_out/r4z_parity_wide.jsonl timeout 3000 python -m pytest tests/test_gpu_scale.py -m gpu -q -k test_wide_campaign 2>&1 | tail -3 > gpurun_out/r4z_wide.txt
cat gpurun_out/r4z_wide.txt; wc -l gpurun_out/r4z_parity_wide.jsonl
