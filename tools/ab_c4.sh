#!/bin/bash
# A/B the C4 (g = 8, 128k) decode attend of several liboscar builds (run on the GPU box)
cd "$(dirname "$0")/.."
for lib in "$@"; do
  if [ "$lib" = default ]; then unset OSCAR_LIB; else export OSCAR_LIB=$lib; fi
  python bench.py --c4-only --steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', 'attend_us=%.1f' % d['attend_us'], 'frac=%.3f' % d['roofline']['frac'])"
done
