set -u
o=gpurun_out/${TAG:-g3pp}; mkdir -p $o
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
PROFILE=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/p7_launches.csv python tools/bench3.py poisson7 255 point > $o/ncu.log 2>&1
PROFILE=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/a7_launches.csv python tools/bench3.py aniso7 255 planes >> $o/ncu.log 2>&1
python tools/launches.py $o/p7_launches.csv 100000 1 | head -12
python tools/launches.py $o/a7_launches.csv 100000 1 | head -14
