for lib in paper_2103_00959_b200/libgsp.so variants/*.so; do
  echo "$lib $(GSP_LIB=$PWD/$lib timeout 200 python tools/gat_probe.py C3 2>&1 | tail -1)"
done
