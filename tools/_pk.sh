for v in 99999999 2048 512 128 64; do
  echo "MINK=$v"; EXAGEO_PANEL_CUTLASS_MINK=$v python tools/quick_timing.py 5000 10000 40000 100000 2>&1 | sed 's/ll=.*total=/total=/'
done
