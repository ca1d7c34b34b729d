set -u
o=gpurun_out/l; mkdir -p $o
for rep in 1 2; do VARIANTS="base sum2" WLS="aniso:4095 poisson:8191" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err; done
timeout 300 python bench.py --steps 20 --warmup 5 > $o/bench.json 2>$o/bench.err
python -c "import json; d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]); s=d.get('solve') or {}; print(d['ms_per_step'], s.get('setup_ms'), s.get('setup_device_ms'))"
