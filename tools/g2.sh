mkdir -p gpurun_out
cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/step_cost step_cost.cu && /tmp/step_cost > ../../gpurun_out/g2_stepcost.txt 2>&1; cd ../..
timeout 300 python tools/stencil_abl.py > gpurun_out/g2_abl.txt 2>&1
timeout 300 python tools/stencil_exp.py --tasks > gpurun_out/g2_tasks.txt 2>&1
timeout 300 python tools/stencil_exp.py > gpurun_out/g2_bands.txt 2>&1
