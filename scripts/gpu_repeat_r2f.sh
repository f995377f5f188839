# race checks for r02e/f's a10 fast fire and bit-sliced class recount: repeated runs identical
cd $GRAFT_REPO_ROOT
R=scripts/repeat_check.py
python $R c5 15
python $R c5 15 class_book=0
python $R c5 10 class_wmax=1.0
python $R c5 10 shards=2 T=50.0
python $R c5 20 "dims=(2048,2048)" max_ctas=7 T=60.0
python $R c5 20 "dims=(2048,2048)" class_book=0 max_ctas=3 T=60.0
python $R c3 10 early_reject=1 T=10.0
python $R c3 10 early_reject=1 class_book=1 class_wmax=0.2 T=10.0
python $R c3 20
