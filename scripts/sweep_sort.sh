for c in 0 1 2 3 4 5; do HB_SORT_CFG=$c python scripts/sweep_sort.py run; done
