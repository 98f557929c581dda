#!/bin/bash
# A/B the attend path of several liboscar builds on the C2 decode workload (run on the GPU box):
# tools/ab_attend.sh build_ab/liboscar_a.so build_ab/liboscar_b.so ...   (default lib = "default")
cd "$(dirname "$0")/.."
for lib in "$@"; do
  if [ "$lib" = default ]; then unset OSCAR_LIB; else export OSCAR_LIB=$lib; fi
  python bench.py --layers 8 --steps 20 --warmup 5 --no-extras 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$lib', 'attend_us=%.2f' % r['avg_launch_us'], 'frac=%.3f' % r['frac'], 'step_ms=%.3f' % d['ms_per_step'])"
done
