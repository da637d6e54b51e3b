out=gpurun_out
tag=${1:-g4}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $out/gpu_tests_$tag.log 2>&1; echo "pytest rc=$?" >> $out/gpu_tests_$tag.log
timeout 600 python tools/probe_perf.py 28 32 > $out/probe_$tag.log 2>&1
QG_N=28 QG_BLOCKS=1000 QG_REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_pass -s 12 -c 1 -o $out/prof28r_$tag python tools/prof_one.py > $out/ncu28r_$tag.log 2>&1
echo done
