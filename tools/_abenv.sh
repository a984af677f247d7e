# interleaved A/B of environment knobs (same box, same library): sequential / greedy latency
# usage: NET=inception_v3 bash tools/_abenv.sh "IOS_DEEP_RING=0" "IOS_DEEP_RING=1 IOS_MIN_CPS=8" ...
NET=${NET:-inception_v3}
for r in 1 2; do
  for v in "$@"; do
    echo -n "[$v] "; env $v timeout 150 ${CMD:-python tools/seq_greedy.py --net $NET --steps 50} 2>&1 | tail -1
  done
done
