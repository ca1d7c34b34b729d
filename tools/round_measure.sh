#!/bin/bash
# One GPU call's worth of round measurements (run under gpurun from the repo root):
# every BASELINE config through bench.py, plus the line-relaxation cycle's launch list.
set -u
out=gpurun_out/rm
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1
run() { timeout 400 python bench.py "$@" >> $out/configs.jsonl 2>> $out/configs.err; }
run --config poisson33 --steps 200
run --config checker1025 --steps 100 --pcg 1
run --config aniso4097 --steps 30 --e2e-steps 2
run --config aniso4097 --relax yline --steps 30 --e2e-steps 2 --pcg 1
run --config aniso4097 --relax altline --steps 30 --e2e-steps 2 --no-cpu-baseline
run --config checker4096 --steps 50 --e2e-steps 2 --pcg 1
run --config poisson8193 --steps 200
run --config poisson8193 --steps 200 --no-cpu-baseline --e2e-steps 0 --unfused
run --config poisson8193 --steps 40 --no-cpu-baseline --e2e-steps 0 --nrhs 8
run --config checker4096 --steps 40 --no-cpu-baseline --e2e-steps 0 --nrhs 4 --pcg 1
N=4095 WL=aniso NCYC=1 RELAX=2 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/yline_launches.csv python tools/profile_cycle.py > $out/ncu.log 2>&1
N=8191 WL=poisson NCYC=2 RELAX=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/cycle_launches.csv python tools/profile_cycle.py >> $out/ncu.log 2>&1
N=8191 WL=poisson NCYC=1 NRHS=8 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/block8_launches.csv python tools/profile_cycle.py >> $out/ncu.log 2>&1
