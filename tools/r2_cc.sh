set -u
o=gpurun_out/cc; mkdir -p $o
timeout 1200 python -m pytest tests -q -m gpu > $o/gputest.txt 2>&1; tail -1 $o/gputest.txt
timeout 900 python bench.py > $o/bench.json 2> $o/bench.err
python -c "import json; d=json.loads(open('$o/bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['cycle_dram_frac'], d['clocks'], d['e2e']['value'], d['solve']['setup_device_ms'])"
run() { timeout 600 python bench.py "$@" >> $o/configs.jsonl 2>> $o/configs.err; }
run --config poisson33 --steps 200 --no-cpu-baseline
run --config checker1025 --steps 100 --pcg 1 --no-cpu-baseline
run --config aniso4097 --steps 30 --e2e-steps 2 --no-cpu-baseline
run --config aniso4097 --relax yline --steps 30 --e2e-steps 2 --pcg 1 --no-cpu-baseline
run --config checker4096 --steps 50 --e2e-steps 2 --pcg 1 --no-cpu-baseline
run --config poisson8193 --steps 40 --no-cpu-baseline --e2e-steps 0 --nrhs 8
run --config poisson8193 --steps 40 --no-cpu-baseline --e2e-steps 0 --unfused
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
N=8191 WL=poisson NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/cycle_launches.csv python tools/profile_cycle.py > $o/ncu.log 2>&1
N=1023 WL=checker NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/cycle1023_launches.csv python tools/profile_cycle.py >> $o/ncu.log 2>&1
N=4095 WL=aniso NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/cycle4095_launches.csv python tools/profile_cycle.py >> $o/ncu.log 2>&1
