mkdir -p gpurun_out
for v in cur nostore notmem; do
  if [ $v = cur ]; then L=""; else L=paper_2011_01302_b200/build/libios_$v.so; fi
  IOS_LIB=$L python tools/trace_stage.py inception_v3 "[([5],0),([19,22],0),([98,101,102,105],0)]" > gpurun_out/s3j_trace_$v.log 2>&1
done
for r in 1 2; do for v in cur nostore notmem; do
  if [ $v = cur ]; then L=""; else L=paper_2011_01302_b200/build/libios_$v.so; fi
  echo -n "$v "; IOS_LIB=$L timeout 200 python tools/time_schedule.py profiles/r2_sched_inception.json --steps 100 2>&1 | tail -1
done; done
