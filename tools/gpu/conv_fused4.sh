for i in 1 2 3 4; do ONLY=fused timeout 20 python tools/probe_conv_fused.py 256 > /tmp/o.txt 2>&1; echo "exit $? $(tail -1 /tmp/o.txt)"; done
for nb in 4 8 64 256; do timeout 40 python tools/probe_conv_fused.py $nb 2>&1 | tail -1; done
for shape in "32 32 20 30" "64 32 56 56" "100 64 16 24" "32 64 12 20"; do timeout 60 python tools/probe_conv_fused.py 4 $shape 2>&1 | tail -1; done
B200_CONV_STATS=1 ONLY=fused timeout 60 python tools/probe_conv_fused.py 256 2>&1 | tail -2
