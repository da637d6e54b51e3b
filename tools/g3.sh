out=gpurun_out
tag=${1:-g3}
QG_N=28 QG_BLOCKS=1000 QG_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_pass -s 12 -c 1 -o $out/prof28r_$tag python tools/prof_one.py > $out/ncu28r_$tag.log 2>&1
QG_N=28 QG_KIND=qft QG_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_pass -s 2 -c 1 -o $out/prof28q_$tag python tools/prof_one.py > $out/ncu28q_$tag.log 2>&1
echo done
