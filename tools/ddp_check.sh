timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 3 --warmup 3 --rows 2000000 --no-cpu-baseline > gpurun_out/ddp1.json 2> gpurun_out/ddp1.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:linear -c 2 --csv python tools/bench_configs.py --only 4a > gpurun_out/lin_times.csv 2>&1
python tools/bench_configs.py --only 4a,3 > gpurun_out/cfg.log 2>&1
timeout 300 python -m pytest tests/test_gpu_linear_cert.py -q 2>&1 | tail -1 >> gpurun_out/cfg.log
