#!/bin/bash
# Round-2 measurement batch (one gpurun call): tests, smoke, bench lines of every config, the ncu
# launch list of exactly the benched Inception schedule + one --set full capture of its first stages.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/f2_gpu_tests.log 2>&1; tail -1 gpurun_out/f2_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --save-schedule gpurun_out/f2_sched_inception_v3.json > gpurun_out/f2_bench_inception_v3.log 2>&1
tail -1 gpurun_out/f2_bench_inception_v3.log | cut -c1-300
ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/f2_ncu_launches_inception.csv python tools/ncu_run.py --schedule gpurun_out/f2_sched_inception_v3.json > gpurun_out/f2_ncu_run.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ios_stage -c 3 -f -o gpurun_out/f2_stage_full python tools/ncu_run.py --schedule gpurun_out/f2_sched_inception_v3.json > gpurun_out/f2_ncu_full.log 2>&1
for n in fig2 squeezenet randwire_ws_small; do
  timeout 1500 python bench.py --net $n --steps 100 --warmup 10 --cpu-sample-s 5 --save-schedule gpurun_out/f2_sched_$n.json > gpurun_out/f2_bench_$n.log 2>&1
  tail -1 gpurun_out/f2_bench_$n.log | cut -c1-200
done
for b in 8 32 128; do
  timeout 900 python bench.py --net squeezenet --batch $b --steps 50 --warmup 5 --cpu-sample-s 2 > gpurun_out/f2_bench_squeezenet_b$b.log 2>&1
  tail -1 gpurun_out/f2_bench_squeezenet_b$b.log | cut -c1-200
done
timeout 3600 python bench.py --net nasnet_a_large --steps 50 --warmup 5 --cpu-sample-s 5 --latency-cache /tmp/f2_lc_nasnet.txt --save-schedule gpurun_out/f2_sched_nasnet_a_large.json > gpurun_out/f2_bench_nasnet_a_large.log 2>&1
tail -1 gpurun_out/f2_bench_nasnet_a_large.log | cut -c1-300
