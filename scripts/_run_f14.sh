for tb in 0 1 2 4 8; do FKB_SPMM_TMA=$tb timeout 300 python scripts/spmm_time.py c2 2>&1 | tail -1; done
FKB_SPMM_TMA=4 timeout 300 python scripts/spmm_time.py c4 2>&1 | tail -1
timeout 300 python scripts/spmm_time.py c4 2>&1 | tail -1
