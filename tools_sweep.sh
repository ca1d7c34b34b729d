cd $GRAFT_REPO_ROOT
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cycle_launches.csv python tools_profile_cycle.py > /dev/null 2>&1
WL=aniso N=4095 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/cycle_launches_aniso.csv python tools_profile_cycle.py > /dev/null 2>&1
ls -la gpurun_out/*.csv
