#!/bin/bash
# KNN (real, fp16 path) timing under pipeline variants: python tools/knn_real_bench.py n d K rows
N=${1:-400000}
shift
for v in "$@"; do
  echo "== $v"; env $v python tools/knn_real_bench.py $N 100 10 3 2>&1 | grep iter | tail -1
done
