#!/bin/bash
# dev helper (GPU box): GPU tests without the slow ones, then compact bench
# lines for the configs given as arguments (default: 3).  Extra environment
# (SFB_*, SINCFFT_B200_LIB) passes through.
cd "$(dirname "$0")/.."
[ -z "$NOTEST" ] && python -m pytest tests -m gpu -x -q -k "not slow" 2>&1 | tail -2
for c in ${@:-3}; do
  python bench.py --no-cpu --config $c --steps ${STEPS:-30} 2>/dev/null | python3 -c "
import sys,json
d=json.loads(sys.stdin.readline())
print('config $c', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d.get('stage_ms',{}).items()}, 'e2e', round(d['e2e']['ms_per_step'],3))"
done
