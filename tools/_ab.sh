# interleaved A/B of library builds (same box): sequential / greedy latency of a network
NET=${NET:-inception_v3}
for r in 1 2 3; do
  for v in ${VARIANTS:-cur r1}; do
    if [ $v = cur ]; then L=""; else L=paper_2011_01302_b200/build/libios_$v.so; fi
    echo -n "$v "; IOS_LIB=$L timeout 150 python tools/seq_greedy.py --net $NET --steps 50 2>&1 | tail -1
  done
done
