# Measured the direct-load fused-conv converter (B200_CONV_FUSED_RAW / B200_CONV_PFD knobs),
# a variant that was not kept; with it removed both arms run the TMA raw ring.
timeout 600 python -m pytest tests/test_gpu_conv_fused.py -x -q > gpurun_out/conv_direct_tests.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/conv_direct_tests.log
for nb in 8 32 128 256; do
  echo "nb $nb direct:"; timeout 60 python tools/probe_conv_fused.py $nb 2>&1 | tail -1
  echo "nb $nb raw:"; B200_CONV_FUSED_RAW=1 timeout 60 python tools/probe_conv_fused.py $nb 2>&1 | tail -1
done
for pfd in 0 1 3; do echo "pfd $pfd"; B200_CONV_PFD=$pfd timeout 60 python tools/probe_conv_fused.py 256 2>&1 | tail -1; done
for no in 1 3; do echo "nout $no"; B200_CONV_NOUT=$no timeout 60 python tools/probe_conv_fused.py 256 2>&1 | tail -1; done
