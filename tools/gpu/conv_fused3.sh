for v in "B200_CONV_NOUT=2" "B200_CONV_NOUT=1" "B200_CONV_NOUT=0"; do
  echo "== $v"; env $v timeout 40 python tools/probe_conv_fused.py 8 || echo "exit $?"
done
