set -u
o=gpurun_out/${TAG:-g3r}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu3d.py -q -x > $o/test.log 2>&1; tail -2 $o/test.log
for v in "8,32" "4,32" "4,64" "8,64" "8,128" "16,32" "16,64"; do
  BMG3_RB=$v timeout 300 python bench.py --config 3d-poisson7-255 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/rb_$v.json 2>> $o/err.log
  python -c "import json,sys; d=json.load(open('$o/rb_$v.json')); print('$v', round(d['ms_per_step'],3), round(d['roofline']['sweep_ms'],4), round(d['roofline']['frac'],3))"
done
