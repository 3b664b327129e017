# Final round-1 capture of the current build (run on the GPU box from the repo root).
# Each ncu command runs only after the same bench command exited 0 without ncu.
set -x
python bench.py > gpurun_out/bench_r01i.json 2> gpurun_out/bench_r01i.err || exit 1
python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/final_tests.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01i.csv python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/ncu_launch_i.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_add$" -s 5 -c 1 -o gpurun_out/prof_r01i_add python bench.py --steps 6 --warmup 3 --no-secondary > gpurun_out/ncu_full_i.log 2>&1
ncu -i gpurun_out/prof_r01i_add.ncu-rep --page raw --csv > gpurun_out/prof_r01i_add.raw.csv 2>/dev/null
ls -la gpurun_out
