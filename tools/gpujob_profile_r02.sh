# Round-2 profile: bench line, ncu launch list, ncu --set full of the b1 and
# b16 decode kernels, every config's timing (tools/config_sweep.py).
set -u
mkdir -p gpurun_out
bash tools/profile_round.sh r02
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_step -s 3 -c 1 \
    -o gpurun_out/decode_r02_b16 python tools/perf_probe.py --batch 16 --ncu > gpurun_out/ncu_full_r02_b16.log 2>&1
echo "ncu b16 rc=$?"
timeout 900 python tools/config_sweep.py --steps 40 --out gpurun_out/configs_r02.json > gpurun_out/configs_r02.log 2>&1
echo "sweep rc=$?"; tail -20 gpurun_out/configs_r02.log
