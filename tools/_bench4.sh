for rep in 3 10; do for n in fig2 squeezenet inception_v3; do for k in 1 2; do
  IOS_SEARCH_REPS=$rep timeout 900 python bench.py --net $n --steps 100 --warmup 10 --cpu-sample-s 0.1 > /tmp/b.log 2>&1
  tail -1 /tmp/b.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('reps $rep $n', d['value'], d['sequential_ms'], d['greedy_ms'], d['search_s'])"
done; done; done
