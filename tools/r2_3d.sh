set -u
o=gpurun_out/${TAG:-g3p}; mkdir -p $o
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1
for a in "poisson7 255 point" "aniso7 255 planes" "checker27 255 point" "checkeraniso7 255 planes" "poisson7 511 point"; do
  timeout 300 python tools/bench3.py $a >> $o/bench3.jsonl 2>> $o/bench3.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
PROFILE=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/p7_launches.csv python tools/bench3.py poisson7 255 point > $o/ncu.log 2>&1
PROFILE=1 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics $M --csv --log-file $o/a7_launches.csv python tools/bench3.py aniso7 255 planes >> $o/ncu.log 2>&1
