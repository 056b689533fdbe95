# quick GPU pass: smoke (bail out fast), parity, bench fused vs split
set -x
timeout 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo smoke_rc=$rc
cat gpurun_out/smoke.log | tail -5
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu --timeout 120 -x > gpurun_out/pytest_parity.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_parity.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_fused.log 2>&1; echo bench_rc=$?
tail -2 gpurun_out/bench_fused.log | cut -c1-2500
