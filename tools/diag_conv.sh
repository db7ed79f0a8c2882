# MMA-thread phase clocks (DBG 16 | 8) with and without epilogue work (DBG 1)
for d in 24 25; do
  echo "== fp8 56x56 3x3 DBG=$d"; NEOB200_DBG=$d python tools/dbg_clk.py --mode fp8 --n 64 --c 64 --k 64 --hw 56 --r 3 --iters 1 2>&1 | tail -6
  echo "== bf16 14x14 3x3 DBG=$d"; NEOB200_DBG=$d python tools/dbg_clk.py --mode bf16 --n 64 --c 256 --k 256 --hw 14 --r 3 --iters 1 --tile '{"tile_w": 14, "tile_h": 9, "tile_img": 1, "tile_n": 256, "slices_per_stage": 1, "stages": 3}' 2>&1 | tail -6
done
