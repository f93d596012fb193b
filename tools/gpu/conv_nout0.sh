for cfg in "B200_CONV_NOUT=0 B200_CONV_RAW=4" "B200_CONV_NOUT=0 B200_CONV_RAW=8" "B200_CONV_NOUT=1 B200_CONV_RAW=4" "B200_CONV_NOUT=2 B200_CONV_RAW=4"; do
echo "== $cfg"; env $cfg B200_CONV_STATS=1 ONLY=fused timeout 60 python tools/probe_conv_fused.py 256 2>&1 | grep stats
env $cfg timeout 60 python tools/probe_conv_fused.py 256 2>&1 | tail -1
done
