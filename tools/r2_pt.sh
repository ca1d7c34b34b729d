set -u
o=gpurun_out/${TAG:-g3t}; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu3d.py -q -x > $o/test.log 2>&1; tail -2 $o/test.log
for c in 3d-aniso7-255 3d-checkeraniso7-255 3d-poisson7-255 3d-checker27-255; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/$c.json 2>> $o/err.log
  python -c "import json,sys; d=json.load(open('$o/$c.json')); print('$c', round(d['ms_per_step'],3), d['kernels_per_cycle'], round(d['roofline']['sweep_ms'],4), round(d['roofline']['frac'],3), d['solve']['iterations'])"
done
BMG3_NO_PTAIL=1 timeout 300 python bench.py --config 3d-aniso7-255 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/noptail.json 2>> $o/err.log
python -c "import json,sys; d=json.load(open('$o/noptail.json')); print('no ptail', round(d['ms_per_step'],3), d['kernels_per_cycle'])"
