#!/bin/bash
# A/B timing of two builds of libsphb.so in ONE gpurun call (boxes differ by
# several percent, so A and B must share a box):
#   make -C paper_2405_05155_b200/csrc OUT=../libsphb_b.so OBJDIR=../../build/obj_b EXTRA=-D<flag>
#   bash scripts/ab_wc.sh [n_side] [kernel] [reps]
N=${1:-256}; K=${2:-1.6h}; R=${3:-3}
for r in $(seq $R); do
  for v in a b; do
    lib=""; [ $v = b ] && lib=$PWD/paper_2405_05155_b200/libsphb_b.so
    echo "$v $(SPHB_LIB=$lib python scripts/tune_wc.py --one --n-side $N --kernel $K 2>&1 | tail -1)"
  done
done
