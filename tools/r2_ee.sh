set -u
o=gpurun_out/ee; mkdir -p $o
for rep in 1 2; do for v in kc32 kc51 kc26 kc64; do
  BMG_LIB=$PWD/tools/vlib/libbmg_$v.so timeout 300 python bench.py --config 3d-poisson7-255 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $o/b_$v.json 2>$o/b_$v.err
  python -c "import json; d=json.loads(open('$o/b_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), d['roofline'].get('launch_ms'), d['roofline'].get('frac'))"
done; done
BMG_LIB=$PWD/tools/vlib/libbmg_kc51.so timeout 900 python -m pytest -q -x tests/test_gpu3d.py > $o/test.log 2>&1; tail -1 $o/test.log
