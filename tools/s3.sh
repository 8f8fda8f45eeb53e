LEMGPU_EAGER=1 timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:k_mfd_tiles -s 6 -c 2 -o gpurun_out/ncu_mfdq python bench.py --workload dem10000mfd --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_mfdq.log 2>&1
tail -2 gpurun_out/ncu_mfdq.log
