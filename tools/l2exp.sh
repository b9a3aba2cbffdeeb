set -x
for CH in 64 8 4; do
  for PM in 0 64; do
    DREG_L2_PERSIST=$PM DREG_L2_VERBOSE=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --chunk $CH --pairs-per-gpu 64 2>&1 | grep -o '"value": [0-9.]*\|L2 persist.*' | head -3
  done
done
