#!/bin/bash
# A/B timing of builds of libsphb.so in ONE gpurun call (boxes differ by
# several percent, so the variants must share a box).  Variant x is
# paper_2405_05155_b200/libsphb_x.so ("a" = the default build):
#   make -C paper_2405_05155_b200/csrc OUT=../libsphb_b.so OBJDIR=../../build/obj_b EXTRA=-D<flag>
#   bash scripts/ab_wc.sh [n_side] [kernel] [reps] [variants, default "a b"]
N=${1:-256}; K=${2:-1.6h}; R=${3:-3}; V=${4:-a b}
for r in $(seq $R); do
  for v in $V; do
    lib=""; [ $v != a ] && lib=$PWD/paper_2405_05155_b200/libsphb_$v.so
    echo "$v $(SPHB_LIB=$lib python scripts/tune_wc.py --one --n-side $N --kernel $K 2>&1 | tail -1)"
  done
done
