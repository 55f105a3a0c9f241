#!/bin/bash
# time apply_F for c2 across stagger settings
for s in 0 500 1000 2000; do for m in 3 6; do
  echo "stagger=$s mod=$m: $(PIT_STAGGER=$s PIT_STAGGER_MOD=$m python tools/time_ops.py c2 5 2>&1 | grep apply_F)"
done; done
