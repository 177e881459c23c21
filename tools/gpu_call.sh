timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 900 python tools/p_ladder.py 1000000 6 8 10 11 12 13 14 15 > gpurun_out/p_ladder.jsonl 2> gpurun_out/p_ladder.err
cat gpurun_out/p_ladder.jsonl | cut -c1-400
