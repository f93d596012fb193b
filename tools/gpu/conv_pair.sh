for nb in 1 4 8 64 256; do ONLY=fused timeout 30 python tools/probe_conv_fused.py $nb > /tmp/o.txt 2>&1; echo "nb $nb exit $? $(tail -1 /tmp/o.txt)"; done
for nb in 4 64 256; do timeout 60 python tools/probe_conv_fused.py $nb 2>&1 | tail -1; done
B200_CONV_PAIR=0 timeout 60 python tools/probe_conv_fused.py 256 2>&1 | tail -1
B200_CONV_STATS=1 ONLY=fused timeout 60 python tools/probe_conv_fused.py 256 2>&1 | grep stats
for shape in "32 32 20 30" "64 32 56 56" "48 64 16 24"; do timeout 60 python tools/probe_conv_fused.py 4 $shape 2>&1 | tail -1; done
