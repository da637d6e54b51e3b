# usage: bash tools/gpu_prof.sh TAG [N]  -- ncu capture of one random-CX and one QFT fused pass (dev tool)
out=gpurun_out
tag=${1:-p}
n=${2:-28}
QG_N=$n QG_BLOCKS=1000 QG_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_pass -s 12 -c 1 -o $out/prof${n}r_$tag python tools/prof_one.py > $out/ncu${n}r_$tag.log 2>&1
QG_N=$n QG_KIND=qft QG_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_pass -s 2 -c 1 -o $out/prof${n}q_$tag python tools/prof_one.py > $out/ncu${n}q_$tag.log 2>&1
echo done
