set -x
timeout 60 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo smoke_rc=$rc; tail -3 gpurun_out/smoke.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu --timeout 60 -x > gpurun_out/pytest_parity.log 2>&1; echo pytest_rc=$?
tail -25 gpurun_out/pytest_parity.log
for FC in 0 1; do B2P_FC=$FC timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_fc$FC.log 2>&1; tail -c 700 gpurun_out/bench_fc$FC.log; done
