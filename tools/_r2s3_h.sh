mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3h_tests_cur.log 2>&1; tail -2 gpurun_out/s3h_tests_cur.log
IOS_LIB=paper_2011_01302_b200/build/libios_latepdl.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedules.py -q -x -k "not refined and not cluster and not searched" > gpurun_out/s3h_tests_latepdl.log 2>&1; tail -2 gpurun_out/s3h_tests_latepdl.log
for r in 1 2 3; do for v in prev cur latepdl; do
  if [ $v = cur ]; then L=""; else L=paper_2011_01302_b200/build/libios_$v.so; fi
  echo -n "$v "; IOS_LIB=$L timeout 200 python tools/time_schedule.py profiles/r2_sched_inception.json --steps 100 2>&1 | tail -1
  echo -n "$v "; IOS_LIB=$L timeout 200 python tools/seq_greedy.py --net inception_v3 --steps 50 2>&1 | tail -1
  echo -n "$v "; IOS_LIB=$L timeout 300 python tools/seq_greedy.py --net squeezenet --batch 128 --steps 20 2>&1 | tail -1
done; done
timeout 900 python bench.py --net fig2 --steps 100 --warmup 10 --cpu-sample-s 5 > gpurun_out/s3h_bench_fig2.log 2>&1; tail -1 gpurun_out/s3h_bench_fig2.log | cut -c1-150
