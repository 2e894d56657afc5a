#!/bin/bash
# The measurements behind DESIGN.md §7 (run on one B200 through gpurun, from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/reproduce_round1.sh'
# Results land in gpurun_out/repro_*.  Timing rules as in bench.py (CUDA events, L2 flush,
# W >= 3 warm-up steps); every line is also a parity-checked configuration (tests/).
set -u
mkdir -p gpurun_out
out=gpurun_out/repro
# 7.2: per-config throughput (the default line is C2 BILINEAR, SS)
python bench.py > ${out}_bench_c2.json 2>&1
python bench.py --mode nearest --no-cpu-baseline --no-e2e > ${out}_bench_c2_nearest.json 2>&1
for c in 3 4 5 6; do
  python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > ${out}_bench_c$c.json 2>&1
done
python bench.py --config 5 --W 24 --no-cpu-baseline --no-e2e --steps 3 > ${out}_bench_c5w24.json 2>&1
# 7.2: where the time goes (stages switched off; measurement knob, results not used)
for k in 1 2; do
  SPIN_DEBUG_SKIP=$k python bench.py --mode nearest --no-cpu-baseline --no-e2e --steps 10 > ${out}_skip$k.json 2>&1
done
# 7.3: dynamic loop scheduling (15 repetitions where the table says so)
python tools/dls_sweep.py --config 2 --reps 15 > ${out}_dls_c2.jsonl 2>&1
python tools/dls_sweep.py --config 3 --reps 15 --policies STATIC,SS,GSS,FAC,HW --units 0 > ${out}_dls_c3.jsonl 2>&1
python tools/dls_sweep.py --config 3 --reps 5 --P 74 --units 0 > ${out}_dls_c3_p74.jsonl 2>&1
python tools/dls_sweep.py --config 3 --reps 5 --no-sort --units 0 > ${out}_dls_c3_nosort.jsonl 2>&1
python tools/dls_sweep.py --config 5 --reps 15 --units 0 > ${out}_dls_c5w8.jsonl 2>&1
python tools/dls_sweep.py --config 5 --reps 5 --P 74 --units 0 > ${out}_dls_c5w8_p74.jsonl 2>&1
python tools/dls_sweep.py --config 5 --reps 5 --P 296,592 --units 0 > ${out}_dls_c5w8_p296_592.jsonl 2>&1
python tools/dls_sweep.py --config 5 --W 24 --reps 5 --units 0 > ${out}_dls_c5w24.jsonl 2>&1
# 7.3: heterogeneous workers
python tools/dls_sweep.py --config 2 --reps 5 --units 0 --slow 37 --slowdown 4 > ${out}_het_c2.jsonl 2>&1
python tools/dls_sweep.py --config 2 --reps 5 --P 8 --units 0 --slow 2 --slowdown 4 > ${out}_het_c2_p8.jsonl 2>&1
python tools/dls_sweep.py --config 2 --reps 5 --P 8 --units 0 --slow 2 --slowdown 4 --slow-first > ${out}_het_c2_p8_sf.jsonl 2>&1
# 7.3: weighted factoring (WF) and adaptive weighted factoring (AWF)
python tools/dls_sweep.py --config 2 --reps 5 --units 0 --slow 37 --slowdown 4 --policies STATIC,SS,GSS,FAC,WF,AWF > ${out}_het_c2_wf.jsonl 2>&1
python tools/dls_sweep.py --config 2 --reps 5 --P 8 --units 0 --slow 2 --slowdown 4 --policies STATIC,SS,GSS,FAC,WF,AWF > ${out}_het_c2_p8_wf.jsonl 2>&1
python tools/dls_sweep.py --config 3 --reps 5 --units 0 --policies STATIC,SS,FAC,WF,AWF > ${out}_dls_c3_wf.jsonl 2>&1
python tools/dls_sweep.py --config 5 --reps 5 --units 0 --policies STATIC,SS,FAC,WF,AWF > ${out}_dls_c5_wf.jsonl 2>&1
# 7.1/7.2: tensor-core vs packed-fp32 sphere filter, with stages switched off
bash tools/ab_mma.sh > ${out}_ab_mma.txt 2>&1
# §5: seeded fuzz campaigns against the oracle
for seed in 1 2 3 4 5 6 7; do SPIN_FUZZ_SEED=$seed SPIN_FUZZ_CASES=150 python -m pytest tests/test_gpu_parity.py -q -k fuzz > ${out}_fuzz_$seed.log 2>&1; done
# 7.1: isolated pair-test loop variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/hotloop_mma tools/microbench/hotloop_mma.cu && \
  tools/microbench/hotloop_mma > ${out}_hotloop_mma.jsonl 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/hotloop2 tools/microbench/hotloop2.cu && \
  tools/microbench/hotloop2 > ${out}_hotloop2.jsonl 2>&1
echo done
