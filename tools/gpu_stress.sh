mkdir -p gpurun_out
python -m paper_2006_13714_b200.build > /dev/null 2>&1
timeout 1500 python tools/stress.py ${BUDGET:-1200} ${SEED:-77} > gpurun_out/stress_${SEED:-77}.log 2>&1; echo "stress=$?" > gpurun_out/stress_status.txt
