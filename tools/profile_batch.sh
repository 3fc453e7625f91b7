set -x
timeout 300 python tools/bench_scan.py 360 > gpurun_out/c4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
XSCAT_WAVE_PIPES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:wave_walk -s 40 -c 1 -o gpurun_out/walk -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_walk.log 2>&1
XSCAT_WAVE_PIPES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:wave_setup -s 40 -c 1 -o gpurun_out/setup -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_setup.log 2>&1
ls -la gpurun_out
