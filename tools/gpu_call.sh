# final round-2 evidence: bench line, launch lists, HBM tables, p-ladder, C2-C5 configs + C5 sweep
bash tools/profile_r2final.sh > /dev/null 2>&1
timeout 900 python tools/p_ladder.py 1000000 4 5 6 7 8 9 10 11 12 13 14 15 > gpurun_out/r2f_p_ladder.jsonl 2> gpurun_out/r2f_p_ladder.err
timeout 1500 python tools/config_sweep.py configs --steps 10 > gpurun_out/r2f_configs.jsonl 2> gpurun_out/r2f_configs.err
timeout 1500 python tools/config_sweep.py sweep --steps 5 > gpurun_out/r2f_sweep.jsonl 2> gpurun_out/r2f_sweep.err
ls -la gpurun_out/r2f_*
