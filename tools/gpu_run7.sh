set -x
mkdir -p gpurun_out
./tools/bin/coop_launch_probe > gpurun_out/r2_coop_launch_probe.txt 2>&1; cat gpurun_out/r2_coop_launch_probe.txt
timeout 300 python tools/mc_cta_replay.py cfg2 > gpurun_out/r2_mc_cta_cfg2_v5.txt 2>&1; tail -2 gpurun_out/r2_mc_cta_cfg2_v5.txt
for k in k_window_combine_wide k_ms_coop k_window_runs; do
timeout 600 ncu --set full --import-source on --clock-control none -f -k regex:$k -s 300 -c 1 -o gpurun_out/r2_ncu_${k}_frag python tools/prof_replay.py frag 1 > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
