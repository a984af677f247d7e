mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2_gpu_tests1.log 2>&1; tail -15 gpurun_out/r2_gpu_tests1.log
timeout 600 python bench.py --steps 100 --save-schedule gpurun_out/r2_sched_inception.json > gpurun_out/r2_bench1.log 2>&1; tail -1 gpurun_out/r2_bench1.log
timeout 600 python tools/a7_check.py --net inception_v3 > gpurun_out/r2_a7_ios.log 2>&1; tail -3 gpurun_out/r2_a7_ios.log
timeout 600 python tools/a7_check.py --net inception_v3 --schedule seq > gpurun_out/r2_a7_seq.log 2>&1; tail -3 gpurun_out/r2_a7_seq.log
IOS_COOP=1 timeout 600 python bench.py --steps 100 --tune 0 > gpurun_out/r2_bench_coop.log 2>&1; tail -1 gpurun_out/r2_bench_coop.log | cut -c1-200
timeout 600 python bench.py --steps 100 --tune 0 > gpurun_out/r2_bench_nocoop.log 2>&1; tail -1 gpurun_out/r2_bench_nocoop.log | cut -c1-200
