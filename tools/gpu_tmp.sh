tools/latbench > gpurun_out/latbench.txt 2>&1; cat gpurun_out/latbench.txt
