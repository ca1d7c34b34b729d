set -u
o=gpurun_out/t; mkdir -p $o
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $o/smoke.log 2>&1; tail -1 $o/smoke.log
timeout 1200 python -m pytest tests -q -m gpu --durations=5 > $o/gputest.txt 2>&1; tail -1 $o/gputest.txt
timeout 900 python bench.py > $o/bench.json 2> $o/bench.err
python -c "import json; d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['cycle_dram_frac'], d['clocks'], d['solve']['setup_device_ms'], d['gpu_launches'])"
