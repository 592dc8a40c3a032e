#!/bin/bash
# A/B of level-0 kernels: bench level-0 numbers with and without the TMA path
for v in "" "UAAMG_NO_TMA=1"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['config']['level0_kernels']
print('$v', 'value', round(d['value'],4), 'setup', round(d['config']['setup_s'],4), 'solve', round(d['config']['solve_s'],4), ' '.join(f'{n}:{v[\"us_per_launch\"]:.1f}us/{v[\"frac\"]:.3f}' for n,v in k.items()))"
done
