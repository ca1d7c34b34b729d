set -u
o=gpurun_out/e; mkdir -p $o
BMG_LIB=$PWD/tools/vlib/libbmg_tclk.so python tools/tail_clock.py poisson 31 > $o/tclk.txt 2>&1
BMG_LIB=$PWD/tools/vlib/libbmg_tclk.so python tools/tail_clock.py poisson 1023 >> $o/tclk.txt 2>&1
cat $o/tclk.txt
timeout 900 python -m pytest -q -x tests/test_gpu_tail.py tests/test_gpu_parity.py tests/test_gpu_solve.py tests/test_gpu_fullcycle.py tests/test_gpu_dist.py > $o/test.log 2>&1; tail -1 $o/test.log
for c in poisson33 checker1025 poisson8193; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $o/bench_$c.json 2>$o/bench_$c.err
  python -c "import json,sys; d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], (d.get('solve') or {}).get('ms'), d.get('levels',{}).get('tail_ms'), d['roofline'].get('cycle_dram_frac'))"
done
