set -x
python bench.py > gpurun_out/bench_r01f.json 2> gpurun_out/bench_r01f.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01f.csv python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/ncu_launch_f.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_add$" -s 5 -c 1 -o gpurun_out/prof_r01f_add python bench.py --steps 6 --warmup 3 --no-secondary > gpurun_out/ncu_full_f.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_decompress$" -s 3 -c 1 -o gpurun_out/prof_r01f_dec python bench.py --steps 6 --warmup 3 --no-secondary > gpurun_out/ncu_full_fd.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_compress$" -s 3 -c 1 -o gpurun_out/prof_r01f_cmp python bench.py --steps 6 --warmup 3 --no-secondary > gpurun_out/ncu_full_fc.log 2>&1
ls -la gpurun_out
