tools/mma_peaks > gpurun_out/mma_peaks.json 2>&1
