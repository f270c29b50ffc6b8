tools/tf32_layout_test > gpurun_out/tf32_layout.txt 2>&1
