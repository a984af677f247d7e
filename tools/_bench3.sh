mkdir -p gpurun_out
for n in fig2 squeezenet; do
  timeout 900 python bench.py --net $n --steps 100 --warmup 10 --cpu-sample-s 2 --save-schedule gpurun_out/r2_sched_$n.json > gpurun_out/r2_bench_$n.log 2>&1
  tail -1 gpurun_out/r2_bench_$n.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$n', d['value'], d['sequential_ms'], d['greedy_ms'], d['roofline']['frac'])"
  timeout 600 python tools/a7_check.py --net $n > gpurun_out/r2_a7_$n.log 2>&1; tail -2 gpurun_out/r2_a7_$n.log
done
timeout 1200 python bench.py --net randwire_ws_small --steps 100 --warmup 10 --cpu-sample-s 2 --save-schedule gpurun_out/r2_sched_randwire.json > gpurun_out/r2_bench_randwire.log 2>&1
tail -1 gpurun_out/r2_bench_randwire.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('randwire', d['value'], d['sequential_ms'], d['greedy_ms'], d['roofline']['frac'], d['search_s'])"
