# A/B: tools/libvc3_ab_cur.so (cell test, per-decode 2*tol, two-op cell bits)
# vs lib/libvc3_b200.so (hoisted 2*tol, one LOP3); then parity of the new build.
set -x
for i in 1 2 3; do
  python tools/grid_sweep.py tools/libvc3_ab_cur.so paper_2003_02633_b200/lib/libvc3_b200.so
done 2>&1 | tee gpurun_out/ab2_sweep.txt
python -m pytest tests -m gpu -x -q > gpurun_out/ab2_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/ab2_tests.log
python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
VC3_SOAK=28 timeout 600 python -m pytest tests/test_soak.py -x -q -s > gpurun_out/ab2_soak.log 2>&1; echo soak=$?; grep SOAK gpurun_out/ab2_soak.log
