set -u
o=gpurun_out/s; mkdir -p $o
for rep in 1 2; do VARIANTS="base xs xst xr xrs" WLS="aniso:4095" LEGS=down bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err; done
cat $o/sweep.jsonl
