python tools/sp_prof.py save 500 > /dev/null
for f in exp_libs/*.so; do
  echo "== $f"
  PGA_LIB=$f python tools/sp_prof.py load 500
  PGA_LIB=$f timeout 300 python tools/theta_scan.py 1000 -1 cache 2>&1 | tail -1
done
