#!/bin/bash
# FC GEMM tile / split-K sweep (experiments build: CK_TC_BN / CK_TC_BM / CK_TC_SPLITS)
L=paper_1412_4564_b200/_build_exp/libck_exp.so
for layer in fc6 fc7; do
  python tools/conv_layer_bench.py --layers $layer --reps 20 | sed "s/^/default        /"
  for bn in 0 128 64; do for bm in 0 128 256; do for sp in 1 2 3 4 6 8; do
    out=$(CK_TC_BN=$bn CK_TC_BM=$bm CK_TC_SPLITS=$sp python tools/conv_layer_bench.py --lib $L --layers $layer --reps 20 2>&1 | tail -1)
    echo "bn=$bn bm=$bm sp=$sp $out"
  done; done; done
done
