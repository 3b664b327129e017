# ncu captures summarised under profiles/ (run on the GPU box from the repo root).
# Each ncu command runs only after the same bench command exited 0 without ncu.
set -x
python bench.py > gpurun_out/bench_r01f.json 2> gpurun_out/bench_r01f.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01f.csv python bench.py --steps 3 --warmup 3 --no-secondary > gpurun_out/ncu_launch_f.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_add$" -s 5 -c 1 -o gpurun_out/prof_r01f_add python bench.py --steps 6 --warmup 3 --no-secondary > gpurun_out/ncu_full_f.log 2>&1
for k in decompress compress; do
  ncu --set full --clock-control none --import-source on -k "regex:^k_$k\$" -s 3 -c 1 -o gpurun_out/prof_r01f_$k python bench.py --steps 6 --warmup 3 --no-secondary > gpurun_out/ncu_full_$k.log 2>&1
  # keep the raw page only (the 64 MiB copy-back limit)
  ncu -i gpurun_out/prof_r01f_$k.ncu-rep --page raw --csv > gpurun_out/prof_r01f_$k.raw.csv 2>/dev/null
  rm -f gpurun_out/prof_r01f_$k.ncu-rep
done
ls -la gpurun_out
