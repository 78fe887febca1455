#!/bin/bash
# full-size (Amazon2M shape) real KNN under env variants: bash tools/knn_variants_full.sh "VAR=.." ...
for v in "$@"; do
  echo "== $v"; env $v timeout 100 python tools/knn_real_bench.py 2449029 100 10 0 2>&1 | grep iter | tail -1
done
