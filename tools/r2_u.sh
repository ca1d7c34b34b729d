set -u
o=gpurun_out/u; mkdir -p $o
timeout 900 python -m pytest -q -x tests/test_gpu_solve.py tests/test_abi.py > $o/test.log 2>&1; tail -1 $o/test.log
timeout 900 python bench.py > $o/bench.json 2> $o/bench.err
python -c "import json; d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e'], d['clocks'])"
timeout 900 python bench.py --config checker4096 --steps 20 --no-cpu-baseline > $o/bench5.json 2> $o/bench5.err
python -c "import json; d=json.loads(open('$o/bench5.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'])"
