#!/bin/bash
# Same-box A/B with parity: for every tools/ab/*.so, run the parity tests selected by PYTEST_K
# through that build (GB_LIB), then tools/ab.sh timing of the given configs.
#   GPU: gpurun -- 'PYTEST_K="hyb8 or fuzz" bash tools/ab_parity.sh "--config c3" ...'
for lib in tools/ab/*.so; do
  echo "== parity $(basename $lib)"
  GB_LIB=$lib timeout 900 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-hyb8}" 2>&1 | tail -2
done
bash tools/ab.sh "$@"
