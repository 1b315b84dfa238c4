# songs/hour of one lock-step group (tools/songs_bench.py) with its phase split, and a cProfile of the same run
mkdir -p gpurun_out/songs
N=${N:-8}
timeout 600 python tools/songs_bench.py --songs $N --lockstep 8 > gpurun_out/songs/prof.json 2> gpurun_out/songs/prof.err
python -c "import json; d=json.loads(open('gpurun_out/songs/prof.json').read().strip().splitlines()[-1]); print(d['value'], d['wall_s'], d['lockstep_phase_s'])"
timeout 600 python -m cProfile -o gpurun_out/songs/prof.pstats tools/songs_bench.py --songs $N --lockstep 8 > /dev/null 2>&1
python -c "
import pstats; p=pstats.Stats('gpurun_out/songs/prof.pstats'); p.sort_stats('tottime').print_stats(25)" > gpurun_out/songs/prof_top.txt
