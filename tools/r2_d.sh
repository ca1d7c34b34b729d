set -u
o=gpurun_out/d; mkdir -p $o
BMG_LIB=$PWD/tools/vlib/libbmg_tclk.so python tools/tail_clock.py poisson 31 > $o/tclk.txt 2>&1
BMG_LIB=$PWD/tools/vlib/libbmg_tclk.so python tools/tail_clock.py poisson 1023 >> $o/tclk.txt 2>&1
cat $o/tclk.txt
for rep in 1 2; do
VARIANTS="base u192p3 ue1 u192p3e1 u256p4e1" WLS="aniso:4095 poisson:8191" LEGS=down,up,cycle bash tools/sweep.sh >> $o/sweep.jsonl 2>>$o/sweep.err
done
