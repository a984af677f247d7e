#!/bin/bash
# Session-3 check: GPU tests, smoke, Inception bench + ncu launch list of the benched schedule.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s3_gpu_tests.log 2>&1; tail -3 gpurun_out/s3_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --save-schedule gpurun_out/s3_sched_inception_v3.json > gpurun_out/s3_bench_inception_v3.log 2>&1
tail -1 gpurun_out/s3_bench_inception_v3.log
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/s3_ncu_launches_inception.csv python tools/ncu_run.py --schedule gpurun_out/s3_sched_inception_v3.json > gpurun_out/s3_ncu_run.log 2>&1
echo ncu_list $?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:ios_stage -c 3 -f -o gpurun_out/s3_stage_full python tools/ncu_run.py --schedule gpurun_out/s3_sched_inception_v3.json > gpurun_out/s3_ncu_full.log 2>&1
echo ncu_full $?
