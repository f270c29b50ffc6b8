mkdir -p gpurun_out
rm -f gpurun_out/boxf_status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "boxf or ncc" > gpurun_out/pytest_boxf.log 2>&1; echo "pytest=$?" >> gpurun_out/boxf_status.txt
