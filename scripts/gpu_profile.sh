# ncu captures for profiles/: fused receive (C3, 512 frames) and the PN-detection FFT correlation
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:rx_fused -s 3 -c 1 -o gpurun_out/prof_fused python scripts/fused_quick.py C3 512 > gpurun_out/ncu_fused.log 2>&1
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:corr_fft -s 1 -c 1 -o gpurun_out/prof_sync python scripts/sync_quick.py 64 > gpurun_out/ncu_sync.log 2>&1
