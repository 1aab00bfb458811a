# ncu --set full of the fp32 CNN kernels (convolutions, fused BatchNorm): one
# fwd+bwd per ResNet-20 block shape; only the CSV exports come back
LPP_ITERS=1 ncu --set full --clock-control none -k "regex:k_conv|k_wgrad|k_bn_" -c 120 \
    -o /tmp/cnn_full python tools/profile_cnn_kernels.py > gpurun_out/ncu_cnn.log 2>&1
ncu -i /tmp/cnn_full.ncu-rep --page raw --csv > gpurun_out/cnn_full_raw.csv 2>/dev/null
gzip -f gpurun_out/cnn_full_raw.csv
tail -3 gpurun_out/ncu_cnn.log
