# ncu: launch list of a short bench + one full capture of the top kernel ($KREGEX)
set -x
K=${KREGEX:-k_fused}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-latency > gpurun_out/ncu_launch_bench.log 2>&1; echo ncu1_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
  -o gpurun_out/prof_top python bench.py --steps 1 --warmup 1 --batch ${NCU_BATCH:-296} --no-e2e --no-cpu --no-latency > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
tail -3 gpurun_out/ncu_full.log
