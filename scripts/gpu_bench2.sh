mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
