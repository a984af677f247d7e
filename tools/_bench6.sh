for b in 1 8 32 64; do python tools/merge_probe.py --batch $b --stages "8,9,11;17,18,20;97,98,101;99,100;103,104"; done
timeout 900 python bench.py --steps 100 --warmup 10 --cpu-sample-s 2 --save-schedule gpurun_out/r2_sched_inc3.json > gpurun_out/r2_bench_inc3.log 2>&1
tail -1 gpurun_out/r2_bench_inc3.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('inception ios', d['value'], 'dp', d['ios_dp_ms'], 'seq', d['sequential_ms'], 'greedy', d['greedy_ms'], d['roofline']['frac'], d['stage_roofline'])"
for b in 32 128; do
timeout 900 python bench.py --net squeezenet --batch $b --steps 50 --warmup 5 --cpu-sample-s 0.1 > gpurun_out/r2_bench_sq$b.log 2>&1
tail -1 gpurun_out/r2_bench_sq$b.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('squeezenet b$b ios', d['value'], 'dp', d['ios_dp_ms'], 'seq', d['sequential_ms'], 'greedy', d['greedy_ms'], d['roofline'], d['images_per_s'])"
done
