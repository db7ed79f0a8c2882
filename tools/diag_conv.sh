# DenseNet-201 b32 1x1 bottleneck convs with / without the BN-ReLU prologue
for hw in 56 28 14 7; do for c in 256 1024; do
  a=$(python tools/conv_bench.py --n 32 --c $c --k 128 --hw $hw --r 1 --x 32 --y 64 2>&1 | tail -1 | cut -c 1-220)
  b=$(python tools/conv_bench.py --n 32 --c $c --k 128 --hw $hw --r 1 --x 32 --y 64 --prologue 2>&1 | tail -1 | cut -c 1-220)
  echo "hw=$hw c=$c plain: $a"; echo "hw=$hw c=$c pro  : $b"
done; done
