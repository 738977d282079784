P="c1_redrec c3_bird_solve c3_redrec_solve c4_redrec_2048 c4_bird_2048 c4_redrec_h153_1 c4_bird_h153_1 c5_bird_solve_64 c5_bird_solve_1"
python tools/perf_probe.py $P | cut -c1-80
for w in 8; do echo "W=$w"; RECON_GRID_WARPS=$w python tools/perf_probe.py c4_bird_2048 c3_bird_solve c4_redrec_2048 | cut -c1-80; done
python -m pytest tests -m gpu -q -x 2>&1 | tail -1
