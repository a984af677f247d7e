mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests0.log 2>&1; tail -3 gpurun_out/r2_gpu_tests0.log
timeout 600 python bench.py --steps 100 > gpurun_out/r2_bench0.log 2>&1; tail -1 gpurun_out/r2_bench0.log
timeout 600 python tools/schedule_report.py --net inception_v3 --trace 8 > gpurun_out/r2_sched0.log 2>&1; tail -5 gpurun_out/r2_sched0.log
