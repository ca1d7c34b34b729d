set -u
o=gpurun_out/${TAG:-g3tma}; mkdir -p $o
BMG3_RB=t timeout 900 python -m pytest tests/test_gpu3d.py -q -x > $o/test.log 2>&1; tail -2 $o/test.log
for v in t 4,32; do
  BMG3_RB=$v timeout 300 python bench.py --config 3d-poisson7-255 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/rb_$v.json 2>> $o/err.log
  python -c "import json,sys; d=json.load(open('$o/rb_$v.json')); print('$v', round(d['ms_per_step'],3), round(d['roofline']['sweep_ms'],4), round(d['roofline']['frac'],3))"
done
BMG3_RB=t timeout 600 ncu --set full --clock-control none -k regex:k3_rb7t -c 1 -o $o/rb7t_full python tools/bench3.py poisson7 255 point 1 > $o/ncu.log 2>&1
BMG3_RB=t timeout 300 compute-sanitizer --tool memcheck python tools/sanitize3d.py > $o/memcheck.txt 2>&1; tail -1 $o/memcheck.txt
tail -3 $o/err.log
