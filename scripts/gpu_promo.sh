# A/B of the TMA box's L2 promotion (ACA_TMA_PROMO = 256 / 0 / 64 / 128): bench lines of c3/c4/c5
# interleaved twice, DRAM bytes of the c3 / c4 tile kernel per setting (ncu metrics only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-promo}
line() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], '%.4e'%d['value'], round(d['ms_per_step'],2), round(d['roofline']['mean_sweep_ms'],4), d['roofline']['sweeps_per_step'])" $1 "$2"; }
for rep in 1 2; do for C in c3 c4 c5; do for P in 256 0 64 128; do
  ACA_TMA_PROMO=$P timeout 300 python bench.py --config $C --steps 5 --no-cpu --no-e2e > gpurun_out/${TAG}_${C}_${P}_$rep.json 2>/dev/null; line gpurun_out/${TAG}_${C}_${P}_$rep.json "$C promo=$P rep=$rep"
done; done; done
for C in c3 c4; do for P in 256 0 64; do
  ACA_TMA_PROMO=$P timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:tile_grp -s 20 -c 2 --csv python bench.py --config $C --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_${C}_$P.csv 2>/dev/null
  echo "ncu $C $P rc=$?"; grep -E "dram__bytes|gpu__time|lts__" gpurun_out/${TAG}_ncu_${C}_$P.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done; done
