# round 2 (5h): the remaining DLS sweep variants on the final build with clock records: other worker
# counts, the caller-order control, the hardware-scheduler control, uniform brute force
P="STATIC,SS,GSS,FAC"
python tools/dls_sweep.py --config 3 --reps 5 --policies $P --P 74 --units 0 > gpurun_out/r5h_dls_c3_p74.jsonl 2>/dev/null
python tools/dls_sweep.py --config 3 --reps 5 --policies $P --no-sort --units 0 > gpurun_out/r5h_dls_c3_nosort.jsonl 2>/dev/null
python tools/dls_sweep.py --config 3 --reps 5 --policies STATIC,HW --units 0 > gpurun_out/r5h_dls_c3_hw.jsonl 2>/dev/null
python tools/dls_sweep.py --config 5 --reps 5 --policies $P --P 74,296,592 --units 0 > gpurun_out/r5h_dls_c5w8_p.jsonl 2>/dev/null
python tools/dls_sweep.py --config 2 --reps 15 --policies $P > gpurun_out/r5h_dls_c2.jsonl 2>/dev/null
wc -l gpurun_out/r5h_dls_*.jsonl
