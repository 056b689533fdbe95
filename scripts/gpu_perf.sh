# perf iteration: smoke, GPU parity suite, bench (device leg), one ncu full capture of the top kernel
set -x
timeout 90 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo smoke_rc=$rc
tail -3 gpurun_out/smoke.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench.log | cut -c1-400
if [ -n "${PHASE:-}" ]; then timeout 120 python scripts/phase_probe.py > gpurun_out/phase.log 2>&1; cat gpurun_out/phase.log; fi
if [ -n "${NCU:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_fused} -s 1 -c 1 \
    -o gpurun_out/prof_top python bench.py --steps 1 --warmup 1 --batch ${NCU_BATCH:-296} --no-e2e --no-cpu --no-latency > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
fi
