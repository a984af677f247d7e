# cluster split-K: parity test, then A/B of the tiling variants on the benched Inception schedule
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_schedules.py -k cluster -x -q > gpurun_out/s3d_tests.log 2>&1; tail -3 gpurun_out/s3d_tests.log
for r in 1 2; do
  for v in 0 3; do
    echo -n "variant $v untuned: "; IOS_TILE_VARIANT=$v timeout 200 python tools/time_schedule.py profiles/r2_sched_inception.json --tune 0 --steps 100 2>&1 | tail -1
  done
  echo -n "tuned (4 variants): "; timeout 300 python tools/time_schedule.py profiles/r2_sched_inception.json --tune 1 --steps 100 2>&1 | tail -1
done
IOS_TILE_VARIANT=3 IOS_DUMP_PLANS=1 timeout 300 python tools/stage_times.py --schedule profiles/r2_sched_inception.json > gpurun_out/s3d_stage_times_v3.log 2>&1
timeout 300 python tools/stage_times.py --schedule profiles/r2_sched_inception.json > gpurun_out/s3d_stage_times_v0.log 2>&1
