# round 2 (5g): the full DLS experiment on the final build, every line with its clock record
# (tools/dls_sweep.py): C3, C5 W = 8 / 24 with the paper's policies and WF / AWF, and the
# heterogeneous-worker emulation on C2 (37 of 148 workers 4x slower; slow workers requesting first)
P="STATIC,SS,GSS,FAC,WF,AWF"
python tools/dls_sweep.py --config 3 --reps 15 --policies $P > gpurun_out/r5g_dls_c3.jsonl 2> gpurun_out/r5g_dls_c3.err
python tools/dls_sweep.py --config 5 --reps 15 --policies $P > gpurun_out/r5g_dls_c5w8.jsonl 2> gpurun_out/r5g_dls_c5w8.err
python tools/dls_sweep.py --config 5 --W 24 --reps 7 --policies $P > gpurun_out/r5g_dls_c5w24.jsonl 2> gpurun_out/r5g_dls_c5w24.err
python tools/dls_sweep.py --config 2 --reps 15 --policies $P --slow 37 --slowdown 4 > gpurun_out/r5g_dls_hetero_c2.jsonl 2> gpurun_out/r5g_dls_hetero_c2.err
python tools/dls_sweep.py --config 2 --reps 15 --policies $P --slow 37 --slowdown 4 --slow-first > gpurun_out/r5g_dls_hetero_c2_slowfirst.jsonl 2> gpurun_out/r5g_dls_hetero_c2_slowfirst.err
python tools/dls_sweep.py --config 4 --reps 5 --policies STATIC,SS,GSS,FAC --units 0 > gpurun_out/r5g_dls_c4.jsonl 2> gpurun_out/r5g_dls_c4.err
wc -l gpurun_out/r5g_dls_*.jsonl; tail -2 gpurun_out/r5g_dls_c5w8.err
