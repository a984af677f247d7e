mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_schedules.py -k cluster -q > gpurun_out/s3f_tests.log 2>&1; tail -2 gpurun_out/s3f_tests.log
for r in 1 2; do
  for nv in 3 4; do
    echo -n "nv=$nv "; IOS_TUNE_VARIANTS=$nv timeout 300 python tools/time_schedule.py profiles/r2_sched_inception.json --tune 1 --steps 100 2>&1 | tail -1
    echo -n "nv=$nv "; IOS_TUNE_VARIANTS=$nv timeout 300 python tools/seq_greedy.py --net squeezenet --batch 128 --steps 20 --tune 1 2>&1 | tail -1
  done
done
