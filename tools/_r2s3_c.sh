# A/B: base library vs current (time_schedule on the benched Inception schedule, seq/greedy), + plan dump
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in base cur; do
    if [ $v = cur ]; then L=""; else L=paper_2011_01302_b200/build/libios_$v.so; fi
    echo -n "$v "; IOS_LIB=$L timeout 200 python tools/time_schedule.py profiles/r2_sched_inception.json --steps 100 2>&1 | tail -1
    echo -n "$v "; IOS_LIB=$L timeout 200 python tools/seq_greedy.py --net inception_v3 --steps 50 2>&1 | tail -1
  done
done
IOS_DUMP_PLANS=1 python tools/stage_times.py --schedule profiles/r2_sched_inception.json > gpurun_out/s3c_plans.log 2>&1
