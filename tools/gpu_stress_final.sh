# stress runs of the final build: the general mix (incl. 3D, NCC, tcf, heaps) and the dp4a box kernel focus
mkdir -p gpurun_out/stressf; rm -f gpurun_out/stressf/*
timeout 1100 python tools/stress.py 960 4041 > gpurun_out/stressf/stress_4041.log 2>&1; echo "mix=$?" >> gpurun_out/stressf/status.txt
STRESS_FOCUS=box timeout 420 python tools/stress.py 300 4042 > gpurun_out/stressf/stress_box_4042.log 2>&1; echo "box=$?" >> gpurun_out/stressf/status.txt
