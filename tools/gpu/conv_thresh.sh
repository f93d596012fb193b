for nb in 8 16 24 32 48; do timeout 60 python tools/probe_conv_fused.py $nb 2>&1 | tail -1; done
