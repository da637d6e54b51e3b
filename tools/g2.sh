out=gpurun_out
tag=${1:-g2}
timeout 900 python -m pytest tests -m gpu -x -q > $out/gpu_tests_$tag.log 2>&1; echo "pytest rc=$?" >> $out/gpu_tests_$tag.log
timeout 600 python tools/probe_perf.py 28 30 32 > $out/probe_$tag.log 2>&1
echo done
