# the conv / wgrad tile variants (csrc/conv_f32.cu dispatch tables), standalone
for v in 0 1 2 3; do
  echo "== variant $v"
  LPP_CONV_VARIANT=$v LPP_WGRAD_VARIANT=$v python tools/exp_conv_native.py
done
