set -u
o=gpurun_out/o; mkdir -p $o
timeout 1200 python -m pytest -q -x tests/test_gpu3d.py > $o/test.log 2>&1; tail -1 $o/test.log
for c in 3d-poisson7-255 3d-aniso7-255 3d-checker27-255; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_$c.json 2>$o/bench_$c.err
  python -c "import json; d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]); s=d.get('solve') or {}; print('$c', d['ms_per_step'], s.get('setup_ms'))"
done
