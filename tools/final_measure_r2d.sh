#!/bin/bash
# Round-2 final measurement batch (session 3, after the late-PDL / boundary-kernel changes): bench
# lines of every config, the ncu launch list + DRAM traffic of exactly the benched Inception
# schedule, a --set full capture of its first stages, ncu GB/s of memory-bound ops, in-run stage
# times. (Artefacts kept < 64 MiB: gpurun copies back at most that.)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f7_gpu_tests.log 2>&1; tail -1 gpurun_out/f7_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --save-schedule gpurun_out/f7_sched_inception_v3.json > gpurun_out/f7_bench_inception_v3.log 2>&1
tail -1 gpurun_out/f7_bench_inception_v3.log | cut -c1-120
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/f7_ncu_launches_inception.csv python tools/ncu_run.py --schedule gpurun_out/f7_sched_inception_v3.json > gpurun_out/f7_ncu_run.log 2>&1; echo ncu_list $?
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ios_stage -c 6 -f -o gpurun_out/f7_stage_full python tools/ncu_run.py --schedule gpurun_out/f7_sched_inception_v3.json > gpurun_out/f7_ncu_full.log 2>&1; echo ncu_full $?
ncu -i gpurun_out/f7_stage_full.ncu-rep --page raw --csv > gpurun_out/f7_stage_full_raw.csv 2>/dev/null
timeout 600 python tools/stage_times.py --schedule gpurun_out/f7_sched_inception_v3.json > gpurun_out/f7_stage_times_inception.log 2>&1
for n in fig2 squeezenet randwire_ws_small; do
  timeout 1500 python bench.py --net $n --steps 100 --warmup 10 --cpu-sample-s 5 --save-schedule gpurun_out/f7_sched_$n.json > gpurun_out/f7_bench_$n.log 2>&1
  tail -1 gpurun_out/f7_bench_$n.log | cut -c1-120
done
for b in 8 32 128; do
  timeout 900 python bench.py --net squeezenet --batch $b --steps 50 --warmup 5 --cpu-sample-s 2 --save-schedule gpurun_out/f7_sched_squeezenet_b$b.json > gpurun_out/f7_bench_squeezenet_b$b.log 2>&1
  tail -1 gpurun_out/f7_bench_squeezenet_b$b.log | cut -c1-120
done
timeout 600 python tools/stage_times.py --schedule gpurun_out/f7_sched_squeezenet_b128.json > gpurun_out/f7_stage_times_squeezenet_b128.log 2>&1
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/f7_ncu_memops_squeezenet_b128.csv python tools/ncu_ops.py --net squeezenet --batch 128 --ops 2,15,32,38 > /dev/null 2>&1; echo ncu_memops $?
timeout 3600 python bench.py --net nasnet_a_large --steps 50 --warmup 5 --cpu-sample-s 5 --latency-cache /tmp/f7_lc_nasnet.txt --save-schedule gpurun_out/f7_sched_nasnet_a_large.json > gpurun_out/f7_bench_nasnet_a_large.log 2>&1
tail -1 gpurun_out/f7_bench_nasnet_a_large.log | cut -c1-120
du -sh gpurun_out
