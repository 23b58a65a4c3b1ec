#!/bin/bash
# three-accumulator kernel (cta_group 3) vs the default Horner kernel on c4, interleaved
for r in 1 2 3; do
  timeout 300 python scripts/cfg_sustained.py c4 '{}' 12 | sed 's/^/horner /'
  timeout 300 python scripts/cfg_sustained.py c4 '{"cta_group": 3}' 12 | sed 's/^/g3     /'
done
