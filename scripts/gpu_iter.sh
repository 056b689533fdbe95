# quick perf iteration on one box: phase split, device-leg bench (x2), fused parity tests
set -x
timeout 120 python scripts/phase_probe.py 2>&1 | tail -5
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['ms_per_step'], d.get('parity',{}).get('iterations_equal'), d['roofline']['frac'])"; done
timeout 600 python -m pytest tests -q -m gpu -x ${PYTEST_K:--k "parity or fused or shapes"} --timeout 300 2>&1 | tail -3
