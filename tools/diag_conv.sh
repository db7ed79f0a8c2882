T56='{"tile_n": 64, "slices_per_stage": 1, "stages": 2, "weight_stationary": 2}'
T14='{"tile_w": 14, "tile_h": 9, "tile_img": 1, "tile_n": 256, "slices_per_stage": 1, "stages": 3}'
for d in 0 1 4 5; do
  echo "56x56 3x3 DBG=$d: $(NEOB200_DBG=$d python tools/conv_bench.py --n 64 --c 64 --k 64 --hw 56 --r 3 --tile "$T56" 2>&1 | tail -1)"
done
for d in 0 1 4 5; do
  echo "14x14 3x3 DBG=$d: $(NEOB200_DBG=$d python tools/conv_bench.py --n 64 --c 256 --k 256 --hw 14 --r 3 --tile "$T14" 2>&1 | tail -1)"
done
