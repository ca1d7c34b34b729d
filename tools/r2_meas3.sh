#!/bin/bash
# Measurement after the 9-point pairs-per-thread / ring-slack change and the tail rewrite:
# GPU test suite, bench line, configs, cycle launch lists, ncu --set full of the fused legs.
set -u
out=gpurun_out/${TAG:-m3}
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu --durations=5 > $out/gputest.txt 2>&1; tail -1 $out/gputest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $out/bench.json 2> $out/bench.err; tail -c 400 $out/bench.json
run() { timeout 600 python bench.py "$@" >> $out/configs.jsonl 2>> $out/configs.err; }
run --config poisson33 --steps 200 --no-cpu-baseline
run --config checker1025 --steps 100 --pcg 1 --no-cpu-baseline
run --config aniso4097 --steps 30 --e2e-steps 2 --no-cpu-baseline
run --config checker4096 --steps 50 --e2e-steps 2 --pcg 1 --no-cpu-baseline
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
N=8191 WL=poisson NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $out/cycle_launches.csv python tools/profile_cycle.py > $out/ncu.log 2>&1
N=1023 WL=checker NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $out/cycle1023_launches.csv python tools/profile_cycle.py >> $out/ncu.log 2>&1
N=4095 WL=aniso NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $out/cycle4095_launches.csv python tools/profile_cycle.py >> $out/ncu.log 2>&1
N=8191 WL=poisson NCYC=1 RELAX=0 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"k_fused" -c 3 -o $out/fused_full python tools/profile_cycle.py >> $out/ncu.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
