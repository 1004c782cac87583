# ncu evidence on one B200 (each capture after a clean run of the same command):
#   launch lists of one c2/c3/c4 step, --set full of the step's top kernels, the W-block
#   products, the Γ·X column pass and the SpMM.   bash scripts/gpu_ncu.sh TAG
set -x
tag=${1:-r2}
o=gpurun_out
r=/tmp/ncu_reps   # full reports stay on the box (gpurun copies back ≤ 64 MiB); summaries come back
mkdir -p $o $r
P="python scripts/profile.py"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
for c in c2 c3 c4; do
  timeout 300 $P step $c > $o/prof_step_$c.log 2>&1 && \
  timeout 600 ncu --profile-from-start off $M --log-file $o/launches_${c}_$tag.csv $P step $c > /dev/null 2>&1
  python scripts/launch_summary.py $o/launches_${c}_$tag.csv > $o/launches_${c}_$tag.txt 2>&1
done
F="--set full --clock-control none --import-source on --profile-from-start off"
timeout 600 ncu $F -k regex:"k_cap_pcg|k_coldot|k_gemv_rowmajor|k_step_prologue|k_spmv" -o $r/step_c2_$tag -f $P step c2 > $o/ncu_step_c2.log 2>&1
timeout 600 ncu $F -k regex:"k_mean_uq|k_cap_pcg|k_coldot" -o $r/step_c3_$tag -f $P step c3 > $o/ncu_step_c3.log 2>&1
timeout 600 ncu $F -k regex:"k_gemv_rowmajor|k_cap_pcg" -o $r/step_c4_$tag -f $P step c4 > $o/ncu_step_c4.log 2>&1
timeout 300 $P wprod c2 > $o/prof_wprod.log 2>&1 && \
timeout 600 ncu $F -o $r/wprod_c2_$tag -f $P wprod c2 > $o/ncu_wprod.log 2>&1
timeout 300 $P gx c2 592 > $o/prof_gx.log 2>&1 && \
timeout 600 ncu $F -k regex:"k_cols_1|k_rows" -o $r/gx_c2_$tag -f $P gx c2 592 > $o/ncu_gx.log 2>&1
timeout 300 $P gx c4 256 > $o/prof_gx4.log 2>&1 && \
timeout 600 ncu $F -k regex:"k_cols_1|k_rows" -o $r/gx_c4_$tag -f $P gx c4 256 > $o/ncu_gx4.log 2>&1
timeout 300 $P spmm c2 > $o/prof_spmm.log 2>&1 && \
timeout 600 ncu $F -k regex:"k_spmm" -o $r/spmm_c2_$tag -f $P spmm c2 > $o/ncu_spmm.log 2>&1
for k in step_c2 step_c3 step_c4 wprod_c2 gx_c2 gx_c4 spmm_c2; do
  python scripts/ncu_summary.py $r/${k}_$tag.ncu-rep ${k}_$tag > $o/ncu_${k}_$tag.txt 2>&1
done
ls -la $o | tail -30; du -sh $o
for c in c2 c3 c4; do head -14 $o/launches_${c}_$tag.txt; done
