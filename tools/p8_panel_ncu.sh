set -u
mkdir -p gpurun_out
timeout 300 python tools/panel_traffic.py 8 > gpurun_out/p8_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -k regex:filter_step -c 16 --csv python tools/panel_traffic.py 8 > gpurun_out/p8_ncu.csv 2> gpurun_out/p8_ncu.err
echo "rc=$?" >> gpurun_out/p8_ncu.err
CHFSI_SK_HYBRID=0 timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -k regex:filter_step -c 16 --csv python tools/panel_traffic.py 8 > gpurun_out/p8_ncu_hy0.csv 2>> gpurun_out/p8_ncu.err
echo "rc=$?" >> gpurun_out/p8_ncu.err
