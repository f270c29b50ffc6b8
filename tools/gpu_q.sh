mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "${PYTEST_K}" > gpurun_out/pytest_q.log 2>&1; echo "pytest=$?" > gpurun_out/q_status.txt
