mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s3i_tests.log 2>&1; tail -2 gpurun_out/s3i_tests.log
for r in 1 2 3; do for v in prev cur; do
  if [ $v = cur ]; then L=""; else L=paper_2011_01302_b200/build/libios_$v.so; fi
  echo -n "$v "; IOS_LIB=$L timeout 200 python tools/time_schedule.py profiles/r2_sched_inception.json --steps 100 2>&1 | tail -1
  echo -n "$v "; IOS_LIB=$L timeout 200 python tools/seq_greedy.py --net inception_v3 --steps 50 2>&1 | tail -1
  echo -n "$v "; IOS_LIB=$L timeout 200 python tools/seq_greedy.py --net fig2 --steps 100 2>&1 | tail -1
done; done
python tools/trace_stage.py inception_v3 "[([5],0),([56,60,63],0)]" > gpurun_out/s3i_trace.log 2>&1
IOS_LIB=paper_2011_01302_b200/build/libios_fine.so IOS_TRACE_FINE_NAMES=1 python tools/trace_stage.py inception_v3 "[([5],0),([56,60,63],0)]" > gpurun_out/s3i_trace_fine.log 2>&1
timeout 900 python bench.py --net fig2 --steps 100 --warmup 10 --cpu-sample-s 5 > gpurun_out/s3i_bench_fig2.log 2>&1; tail -1 gpurun_out/s3i_bench_fig2.log | cut -c1-120
