set -u
o=gpurun_out/w; mkdir -p $o
timeout 900 python -m pytest -q -x tests/test_gpu_tail.py tests/test_gpu_solve.py tests/test_gpu_parity.py tests/test_gpu_pcg.py > $o/test.log 2>&1; tail -1 $o/test.log
for c in poisson33 checker1025 poisson8193; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $o/bench_$c.json 2>$o/bench_$c.err
  python -c "import json; d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]); s=d.get('solve') or {}; print('$c', d['ms_per_step'], s.get('ms'), d.get('levels',{}).get('tail_ms'))"
done
