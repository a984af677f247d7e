#!/bin/bash
# Round-2 measurement batch (one gpurun call, session 3): GPU tests, smoke, bench lines of every
# config, the ncu launch list of exactly the benched Inception schedule + a --set full capture of
# its stages, ncu DRAM GB/s of memory-bound ops, and a library A/B on SqueezeNet batch 128.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f3_gpu_tests.log 2>&1; tail -1 gpurun_out/f3_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --save-schedule gpurun_out/f3_sched_inception_v3.json > gpurun_out/f3_bench_inception_v3.log 2>&1
tail -1 gpurun_out/f3_bench_inception_v3.log | cut -c1-400
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/f3_ncu_launches_inception.csv python tools/ncu_run.py --schedule gpurun_out/f3_sched_inception_v3.json > gpurun_out/f3_ncu_run.log 2>&1; echo ncu_list $?
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ios_stage -c 40 -f -o gpurun_out/f3_stage_full python tools/ncu_run.py --schedule gpurun_out/f3_sched_inception_v3.json > gpurun_out/f3_ncu_full.log 2>&1; echo ncu_full $?
timeout 600 python tools/stage_times.py --schedule gpurun_out/f3_sched_inception_v3.json > gpurun_out/f3_stage_times_inception.log 2>&1
for n in fig2 squeezenet randwire_ws_small; do
  timeout 1500 python bench.py --net $n --steps 100 --warmup 10 --cpu-sample-s 5 --save-schedule gpurun_out/f3_sched_$n.json > gpurun_out/f3_bench_$n.log 2>&1
  tail -1 gpurun_out/f3_bench_$n.log | cut -c1-250
done
for b in 8 32 128; do
  timeout 900 python bench.py --net squeezenet --batch $b --steps 50 --warmup 5 --cpu-sample-s 2 > gpurun_out/f3_bench_squeezenet_b$b.log 2>&1
  tail -1 gpurun_out/f3_bench_squeezenet_b$b.log | cut -c1-250
done
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/f3_ncu_memops_squeezenet_b128.csv python tools/ncu_ops.py --net squeezenet --batch 128 --ops 2,15,32,38 > /dev/null 2>&1; echo ncu_memops $?
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/f3_ncu_memops_inception_b32.csv python tools/ncu_ops.py --net inception_v3 --batch 32 --ops 4,7,14,39,95,119 > /dev/null 2>&1; echo ncu_memops2 $?
for r in 1 2; do for v in base cur; do
  if [ $v = cur ]; then L=""; else L=paper_2011_01302_b200/build/libios_$v.so; fi
  echo -n "$v sq128 "; IOS_LIB=$L timeout 300 python tools/seq_greedy.py --net squeezenet --batch 128 --steps 20 2>&1 | tail -1
done; done
timeout 3600 python bench.py --net nasnet_a_large --steps 50 --warmup 5 --cpu-sample-s 5 --latency-cache /tmp/f3_lc_nasnet.txt --save-schedule gpurun_out/f3_sched_nasnet_a_large.json > gpurun_out/f3_bench_nasnet_a_large.log 2>&1
tail -1 gpurun_out/f3_bench_nasnet_a_large.log | cut -c1-400
