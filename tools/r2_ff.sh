set -u
o=gpurun_out/ff; mkdir -p $o; rm -f $o/*.jsonl
timeout 900 python -m pytest -q -x tests/test_gpu3d.py > $o/test.log 2>&1; tail -1 $o/test.log
for c in 3d-poisson7-255 3d-poisson7-511 3d-aniso7-255 3d-checker27-255 3d-checkeraniso7-255; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $o/b_$c.json 2>$o/b_$c.err
  tail -1 $o/b_$c.json >> $o/configs3d.jsonl
  python -c "import json; d=json.loads(open('$o/b_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), d['roofline'].get('frac'), (d.get('solve') or {}).get('setup_ms'))"
done
