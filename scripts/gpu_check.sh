# One gpurun pass: smoke, GPU parity suite, bench, ncu launch list + one full capture.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -3 gpurun_out/bench.log
if [ -n "${NCU:-}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-latency > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1_rc=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 \
    -o gpurun_out/prof_k13 python bench.py --steps 1 --warmup 1 --batch 296 --no-e2e --no-cpu --no-latency > gpurun_out/ncu_full_k3.log 2>&1; echo ncu2_rc=$?
fi
cat gpurun_out/smoke.log
