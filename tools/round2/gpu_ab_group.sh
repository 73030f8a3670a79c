cd "$GRAFT_REPO_ROOT"
O=gpurun_out/ab_group; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "grouped or slot_dim" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
for g in 2 4 16; do
  timeout 900 python tools/ab_opts.py --suite s3,set2 --per-cell 2 --kernel-filter tile --esize 4 tile_group=$g > $O/ab_e4_g$g.txt 2>&1; tail -4 $O/ab_e4_g$g.txt
done
timeout 900 python tools/ab_opts.py --suite s2,s3,set2 --per-cell 1 --kernel-filter tile --esize 8 tile_group=4 > $O/ab_e8_g4.txt 2>&1; tail -4 $O/ab_e8_g4.txt
