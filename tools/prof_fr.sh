# ncu captures of the FR divergence kernels (tcgen05 path: compressed and fp32)
set -x
python tools/fr_bench.py > gpurun_out/frb.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:^k_fr_div" -s 2 -c 1 -o gpurun_out/prof_fr_c python tools/fr_bench.py > gpurun_out/ncu_fr.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_fr_div" -s 23 -c 1 -o gpurun_out/prof_fr_f python tools/fr_bench.py > gpurun_out/ncu_fr2.log 2>&1
for r in c f; do ncu -i gpurun_out/prof_fr_$r.ncu-rep --page raw --csv > gpurun_out/prof_fr_$r.raw.csv 2>/dev/null; done
