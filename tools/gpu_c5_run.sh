mkdir -p gpurun_out
(free -g; nproc; nvidia-smi --query-gpu=memory.total,memory.used --format=csv) > gpurun_out/box.txt 2>&1
timeout 600 python -m pytest tests/test_graph_build_gpu.py tests/test_topk.py -q -m gpu -x > gpurun_out/t3_quick.log 2>&1; echo quick rc $?
tail -2 gpurun_out/t3_quick.log
TPA_C5=1 timeout 2400 python -m pytest tests/test_c5.py -q -s -x > gpurun_out/t3_c5.log 2>&1; echo c5 rc $?
tail -20 gpurun_out/t3_c5.log
timeout 1200 python bench.py --config c5 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench c5 rc $?
tail -3 gpurun_out/bench_c5.err
