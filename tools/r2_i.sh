set -u
o=gpurun_out/i; mkdir -p $o
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fullcycle.py tests/test_gpu_dist.py tests/test_gpu_block.py > $o/test.log 2>&1; tail -1 $o/test.log
for c in poisson8193 aniso4097; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $o/bench_$c.json 2>$o/bench_$c.err
  python -c "import json; d=json.loads(open('$o/bench_$c.json').read().strip().splitlines()[-1]); s=d.get('solve') or {}; print('$c', d['ms_per_step'], s.get('setup_ms'), s.get('setup_device_ms'))"
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
N=8191 WL=poisson timeout 300 ncu --metrics $M --clock-control none --csv --log-file $o/setup_launches.csv python tools/profile_setup.py > $o/ncu.log 2>&1
N=4095 WL=aniso timeout 300 ncu --metrics $M --clock-control none --csv --log-file $o/setup_aniso_launches.csv python tools/profile_setup.py >> $o/ncu.log 2>&1
