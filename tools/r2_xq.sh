set -u
o=gpurun_out/r2p; mkdir -p $o
VARIANTS="cur2 xq" WLS="poisson:8191 aniso:4095" bash tools/sweep.sh > $o/sweep.jsonl 2>&1
VARIANTS="cur2 xq" WLS="poisson:8191" bash tools/sweep.sh >> $o/sweep.jsonl 2>&1
