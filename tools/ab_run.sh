# A/B of the decode boundary check in the fused kernels:
#   lib/libvc3_b200.so          cell test in add/axpy, two-conversion test in RK + decompress
#   tools/libvc3_ab_rkcell.so   cell test in the RK stage too
#   tools/libvc3_ab_straddle.so two-conversion test everywhere (previous build)
# then the round's bench line and ncu captures of the default build.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/ab_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
VC3_B200_LIB=$PWD/tools/libvc3_ab_straddle.so python bench.py > gpurun_out/ab_old.json 2>/dev/null
VC3_B200_LIB=$PWD/tools/libvc3_ab_rkcell.so python bench.py > gpurun_out/ab_rkcell.json 2>/dev/null
python bench.py > gpurun_out/bench_r01h.json 2> gpurun_out/bench_r01h.err || exit 1
for f in gpurun_out/ab_old.json gpurun_out/ab_rkcell.json gpurun_out/bench_r01h.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f',round(d['value'],2),{k:round(v['gvec_s'],1) for k,v in d['secondary_kernels'].items()},'rk',round(d['secondary_configs']['C4_rk_stage_icv']['compressed_gvec_s'],2))"; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01h.csv python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/ncu_launch_h.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_add$" -s 5 -c 1 -o gpurun_out/prof_r01h_add python bench.py --steps 6 --warmup 3 --no-secondary > gpurun_out/ncu_full_h.log 2>&1
ncu -i gpurun_out/prof_r01h_add.ncu-rep --page raw --csv > gpurun_out/prof_r01h_add.raw.csv 2>/dev/null
ls -la gpurun_out
