# config-5 songs/hour A/B: modes separated by ';' in MODES
mkdir -p gpurun_out/songs
N=${N:-16}
timeout 300 python -m pytest tests -m gpu -q -k "batched or lockstep" -p no:cacheprovider > gpurun_out/songs/pytest.log 2>&1; echo rc=$? >> gpurun_out/songs/pytest.log
IFS=';' read -ra LIST <<< "${MODES:---concurrent 4;--lockstep 4;--lockstep 8}"
for mode in "${LIST[@]}"; do
  timeout 600 python tools/songs_bench.py --songs $N $mode > gpurun_out/songs/run.json 2> gpurun_out/songs/err.txt
  python -c "import json; d=json.loads(open('gpurun_out/songs/run.json').read().strip().splitlines()[-1]); print('$mode', round(d['value'],1), 'songs/h', round(d['wall_s'],2), 's', d.get('lockstep_phase_s'), [r['trials'] for r in d['per_song']])" >> gpurun_out/songs/ab.txt 2>&1 || tail -3 gpurun_out/songs/err.txt >> gpurun_out/songs/ab.txt
done
