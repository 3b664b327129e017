#!/bin/bash
# Round-2 captures (run under gpurun, one GPU): launch list of a short bench,
# ncu --set full of the fused add in both modes and of compress / decompress.
set -x
python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/prof_bench_plain.json 2> gpurun_out/prof_bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/ncu_launch.log 2>&1
python tools/run_op.py --op add --mode exact > gpurun_out/runop_ex.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_add_as -s 1 -c 1 \
    -o gpurun_out/prof_r02_add_exact python tools/run_op.py --op add --mode exact > gpurun_out/ncu_ex.log 2>&1
python tools/run_op.py --op add --mode contract > gpurun_out/runop_ct.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_add_as -s 1 -c 1 \
    -o gpurun_out/prof_r02_add_contract python tools/run_op.py --op add --mode contract > gpurun_out/ncu_ct.log 2>&1
python tools/run_op.py --op compress > gpurun_out/runop_c.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_compress -s 1 -c 1 \
    -o gpurun_out/prof_r02_compress python tools/run_op.py --op compress > gpurun_out/ncu_c.log 2>&1
python tools/run_op.py --op decompress --mode contract > gpurun_out/runop_d.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_decompress -s 1 -c 1 \
    -o gpurun_out/prof_r02_decompress_contract python tools/run_op.py --op decompress --mode contract > gpurun_out/ncu_d.log 2>&1
ls -la gpurun_out/*.ncu-rep
