mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedules.py -q -x -k "not refined and not cluster and not searched" > gpurun_out/s3l_tests.log 2>&1; tail -1 gpurun_out/s3l_tests.log
for r in 1 2 3; do for v in head cur; do
  if [ $v = cur ]; then L=""; else L=paper_2011_01302_b200/build/libios_$v.so; fi
  echo -n "$v "; IOS_LIB=$L timeout 300 python tools/seq_greedy.py --net randwire_ws_small --steps 50 2>&1 | tail -1
  echo -n "$v "; IOS_LIB=$L timeout 200 python tools/time_schedule.py profiles/r2_sched_inception.json --steps 100 2>&1 | tail -1
done; done
