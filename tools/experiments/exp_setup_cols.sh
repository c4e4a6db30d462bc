# handle creation from device arrays: K_touched by byte marks (current) vs atomicOr bitmap
for lib in "" tools/bin/libdaspmm_oldcols.so "" tools/bin/libdaspmm_oldcols.so; do
  echo "== DASPMM_LIB=$lib"; DASPMM_LIB=$lib timeout 300 python tools/experiments/setup_device_probe.py
done
