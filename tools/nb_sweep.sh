for nb in 8 12 16 20 24 32; do python tools/prof_tc2.py $nb | tail -1; done
python tools/prof_tc2.py 4 ffma | tail -1
