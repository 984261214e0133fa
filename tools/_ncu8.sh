timeout 300 ncu --set full --import-source on --clock-control none -k "regex:oz_gemm" -c 1 --csv --page raw python tools/one_gemm.py 31 64 256 > gpurun_out/ncu8_cfg2_raw.csv 2>/dev/null
timeout 300 ncu --set full --clock-control none -k "regex:oz_gemm" -c 1 --csv --page raw python tools/one_gemm.py 31 16 1024 > gpurun_out/ncu8_cfg3_raw.csv 2>/dev/null
timeout 300 ncu --set full --clock-control none -k "regex:oz_gemm" -c 1 --csv --page raw python tools/one_gemm.py 63 1 2048 > gpurun_out/ncu8_cfg4_raw.csv 2>/dev/null
timeout 300 ncu --set full --clock-control none -k "regex:assemble_c" -c 1 --csv --page raw python tools/one_step.py cfg2 1 > gpurun_out/ncu_asmc_raw.csv 2>/dev/null
