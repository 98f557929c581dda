#!/bin/bash
# Run tools/overhead_probe.py for the default library and every build_ab/liboscar_*.so (GPU box).
cd "$(dirname "$0")/.."
python tools/overhead_probe.py
for lib in build_ab/liboscar_*.so; do
  [ -e "$lib" ] || continue
  OSCAR_LIB=$lib python tools/overhead_probe.py
done
