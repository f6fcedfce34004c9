# A/B: a reference library (abl/libxdrop_head.so) vs the working tree on the default-mode configs
for rep in 1 2 3; do
for lib in "$PWD/abl/libxdrop_head.so" ""; do
  echo "== lib=${lib:-tree}"
  for cfg in ecoli xsweep:100; do
    XDROP_LIB=$lib timeout 300 python tools/sweep_env.py $cfg "XDROP_OCC=3" 2>&1 | tail -1 | cut -c1-75
  done
done
done
