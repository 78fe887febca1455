#!/bin/bash
# quick GPU validation used during development
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -30
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -20
