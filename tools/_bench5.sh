for n in fig2 squeezenet inception_v3 randwire_ws_small; do
  timeout 1500 python bench.py --net $n --steps 100 --warmup 10 --cpu-sample-s 0.1 --save-schedule gpurun_out/r2_sched_ref_$n.json > gpurun_out/r2_bench_ref_$n.log 2>&1
  tail -1 gpurun_out/r2_bench_ref_$n.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$n ios', d['value'], 'dp', d['ios_dp_ms'], 'seq', d['sequential_ms'], 'greedy', d['greedy_ms'], d['refine_stats'], d['search_s'], d['refine_s'])" || tail -5 gpurun_out/r2_bench_ref_$n.log
done
