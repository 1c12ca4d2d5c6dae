# the driver's invocations: defaults, and the reference arm with defaults
O=gpurun_out/r03t; mkdir -p $O
( time timeout 900 python bench.py ) > $O/default.json 2> $O/default.err
( time timeout 900 python bench.py --impl reference ) > $O/ref.json 2> $O/ref.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
