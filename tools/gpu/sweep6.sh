bash tools/gpu/sweep5.sh
SORT=cumulative TOP=70 python tools/profile_sweep.py 128 > gpurun_out/r02_profile_sweep_cum2.txt 2>&1; grep -E "^==|choose_band|band_ok|aff_range|var_range|engine.py.*region|run_tape" gpurun_out/r02_profile_sweep_cum2.txt | cut -c1-150 | sed 's#/tmp/code/arxiv__paper_2307_16080/repo/##'
