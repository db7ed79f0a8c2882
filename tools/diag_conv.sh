# DBG experiments (1: no epilogue work, 4: no operand loads) on the fp8 56x56 3x3
for t in '' '{"tile_w": 56, "tile_h": 2, "tile_img": 1}'; do
for d in 0 1 5; do
  echo "fp8 56x56 3x3 DBG=$d: $(NEOB200_DBG=$d python tools/conv_bench.py --mode fp8 --n 64 --c 64 --k 64 --hw 56 --r 3 --tile "$t" 2>&1 | tail -1)"
done; done
python tools/conv_bench.py --mode fp8 --n 64 --c 64 --k 64 --hw 56 --r 3 --sweep 2>&1 | sort -k2 -n -t'}' | head -12
