# ncu --set full of the fp32 3x3 convolution kernels (standalone, tools/exp_conv_native.py)
ncu --set full --clock-control none --import-source on -k "regex:k_conv3x3|k_wgrad" -c ${NCU_COUNT:-9} \
    -o gpurun_out/conv_full python tools/exp_conv_native.py > gpurun_out/ncu_conv.log 2>&1
ncu -i gpurun_out/conv_full.ncu-rep --page raw --csv > gpurun_out/conv_full_raw.csv 2>/dev/null
ncu -i gpurun_out/conv_full.ncu-rep --page details --csv > gpurun_out/conv_full_details.csv 2>/dev/null
ncu -i gpurun_out/conv_full.ncu-rep --page source --csv --print-source sass -k regex:k_conv3x3 -c 1 > gpurun_out/conv_full_sass.csv 2>/dev/null
tail -3 gpurun_out/ncu_conv.log
