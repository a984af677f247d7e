python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -2
timeout 2400 python tools/schedule_report.py --net nasnet_a_large --latency-cache gpurun_out/lc_nasnet_a_large.txt > gpurun_out/sched_nasnet.txt 2>&1
tail -2 gpurun_out/sched_nasnet.txt
timeout 300 python bench.py --net nasnet_a_large --steps 30 --warmup 3 --cpu-sample-s 0.1 --latency-cache gpurun_out/lc_nasnet_a_large.txt > gpurun_out/bench_nasnet.json 2>&1
timeout 600 python bench.py --net randwire_ws_small --steps 30 --warmup 3 --cpu-sample-s 0.1 --latency-cache gpurun_out/lc_randwire.txt > gpurun_out/bench_randwire.json 2>&1
timeout 300 python bench.py --net squeezenet --steps 30 --warmup 3 --cpu-sample-s 0.1 > gpurun_out/bench_squeezenet.json 2>&1
timeout 300 python bench.py --net inception_v3 --steps 50 --warmup 5 > gpurun_out/bench_inception.json 2>&1
for f in nasnet randwire squeezenet inception; do tail -1 gpurun_out/bench_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['sequential_ms'], d['greedy_ms'], d['search_s'], d['stage_roofline'])"; done
