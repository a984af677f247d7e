#!/bin/bash
# Round-2 measurement batch A (session 3): bench lines of every batch-1 config + the SqueezeNet
# batch sweep, the ncu launch list of exactly the benched Inception schedule + a --set full capture
# of its first stages, ncu DRAM GB/s of memory-bound ops, and a library A/B (split-K workspace).
# (artefacts kept < 64 MiB: gpurun copies back at most that)
mkdir -p gpurun_out
timeout 900 python bench.py --save-schedule gpurun_out/f4_sched_inception_v3.json > gpurun_out/f4_bench_inception_v3.log 2>&1
tail -1 gpurun_out/f4_bench_inception_v3.log | cut -c1-200
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/f4_ncu_launches_inception.csv python tools/ncu_run.py --schedule gpurun_out/f4_sched_inception_v3.json > gpurun_out/f4_ncu_run.log 2>&1; echo ncu_list $?
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ios_stage -c 6 -f -o gpurun_out/f4_stage_full python tools/ncu_run.py --schedule gpurun_out/f4_sched_inception_v3.json > gpurun_out/f4_ncu_full.log 2>&1; echo ncu_full $?
ncu -i gpurun_out/f4_stage_full.ncu-rep --page raw --csv > gpurun_out/f4_stage_full_raw.csv 2>/dev/null
timeout 600 python tools/stage_times.py --schedule gpurun_out/f4_sched_inception_v3.json > gpurun_out/f4_stage_times_inception.log 2>&1
for n in fig2 squeezenet randwire_ws_small; do
  timeout 1500 python bench.py --net $n --steps 100 --warmup 10 --cpu-sample-s 5 --save-schedule gpurun_out/f4_sched_$n.json > gpurun_out/f4_bench_$n.log 2>&1
  tail -1 gpurun_out/f4_bench_$n.log | cut -c1-200
done
for b in 8 32 128; do
  timeout 900 python bench.py --net squeezenet --batch $b --steps 50 --warmup 5 --cpu-sample-s 2 --save-schedule gpurun_out/f4_sched_squeezenet_b$b.json > gpurun_out/f4_bench_squeezenet_b$b.log 2>&1
  tail -1 gpurun_out/f4_bench_squeezenet_b$b.log | cut -c1-200
done
timeout 600 python tools/stage_times.py --schedule gpurun_out/f4_sched_squeezenet_b128.json > gpurun_out/f4_stage_times_squeezenet_b128.log 2>&1
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/f4_ncu_memops_squeezenet_b128.csv python tools/ncu_ops.py --net squeezenet --batch 128 --ops 2,15,32,38 > /dev/null 2>&1; echo ncu_memops $?
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/f4_ncu_memops_inception_b32.csv python tools/ncu_ops.py --net inception_v3 --batch 32 --ops 4,7,14,39,95,119 > /dev/null 2>&1; echo ncu_memops2 $?
for r in 1 2 3; do for v in wsdb cur; do
  if [ $v = cur ]; then L=""; else L=paper_2011_01302_b200/build/libios_$v.so; fi
  echo -n "$v "; IOS_LIB=$L timeout 200 python tools/time_schedule.py gpurun_out/f4_sched_inception_v3.json --steps 100 2>&1 | tail -1
  echo -n "$v "; IOS_LIB=$L timeout 200 python tools/seq_greedy.py --net inception_v3 --steps 50 2>&1 | tail -1
done; done
du -sh gpurun_out
