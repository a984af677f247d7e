python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
python tools/trace_stage.py nasnet_a_large "[([388],0), ([52],0)]" 2>&1 | grep -E "stage|epi done|e:|prologue  "
python tools/trace_stage.py inception_v3 "[([103],0)]" 2>&1 | grep -E "stage|epi done|e:|prologue  "
timeout 300 python tools/op_report.py --net nasnet_a_large --top 30 > gpurun_out/op_report_nasnet.txt 2>&1
timeout 300 python tools/op_report.py --net inception_v3 --top 30 > gpurun_out/op_report_inception.txt 2>&1
timeout 300 python bench.py --net inception_v3 --steps 30 --warmup 5 --cpu-sample-s 0.05 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('inc', d['value'], d['sequential_ms'], d['greedy_ms'])"
