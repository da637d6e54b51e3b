#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 600 python tools/probe_tree.py > $out/p13_tree.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/p13_tree_launches.csv python tools/probe_tree.py > $out/p13_ncu.log 2>&1
echo done
