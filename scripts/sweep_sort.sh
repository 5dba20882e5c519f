for c in ${CFGS:-1 6 7}; do HB_SORT_CFG=$c python scripts/sweep_sort.py run; done
