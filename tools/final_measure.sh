#!/bin/bash
# round-end measurement batch: tests, smoke, bench of every config, ncu launch list + one --set full
# capture (results copied into profiles/ by hand). Latency caches go
# to /tmp on the box: gpurun_out is capped at 64 MiB.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; tail -1 gpurun_out/final_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/final_bench_inception_v3.log 2>&1
for n in fig2 squeezenet randwire_ws_small; do
  timeout 900 python bench.py --net $n --steps 100 --warmup 10 --latency-cache /tmp/final_lc_$n.txt > gpurun_out/final_bench_$n.log 2>&1
done
ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/final_ncu_launches_inception.csv python tools/ncu_run.py --net inception_v3 > gpurun_out/final_ncu_run.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ios_stage -s 10 -c 1 -f -o gpurun_out/final_stage_full python tools/ncu_run.py --net inception_v3 > gpurun_out/final_ncu_full.log 2>&1
timeout 2400 python bench.py --net nasnet_a_large --steps 50 --warmup 5 --cpu-sample-s 5 --latency-cache /tmp/final_lc_nasnet.txt > gpurun_out/final_bench_nasnet_a_large.log 2>&1
du -sh gpurun_out
for f in gpurun_out/final_bench_*.log; do echo $f; tail -n1 $f | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d.get('sequential_ms'), d.get('greedy_ms'), d.get('speedup_vs_sequential'))"; done
