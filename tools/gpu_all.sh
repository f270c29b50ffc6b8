# One GPU round-trip: smoke, GPU parity tests, then the deliverables (bench, reference arm,
# torchrun N=1, ncu launch list, ncu full capture of the matcher).
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" > gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
bash tools/deliverables.sh
cat gpurun_out/deliv_status.txt >> gpurun_out/status.txt
