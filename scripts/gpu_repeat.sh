# race checks: repeated runs of many paths must be identical (scripts/repeat_check.py)
cd $GRAFT_REPO_ROOT
R=scripts/repeat_check.py
python $R c5 15
python $R c3 20 shards=4
python $R c4 20 shards=2
python $R c3 20 early_reject=1
python $R c3 20 early_reject=1 class_book=1 class_wmax=0.05
python $R c4 15 early_reject=1 class_book=1 class_wmax=0.05 beta=0.5 h=0.1 rule=1 init_q=0.05
python $R c2 40 "dims=(1536,1536)" T=10.0
python $R c3 20 lag=2.0 T=5.0
python $R c3 20 checkerboard=-1 T=5.0
python $R c3 20 shards=2 halo_mode=1 T=5.0
python $R c2 30 "tile=(64,64,1)" max_ctas=7
