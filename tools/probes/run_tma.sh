for args in "80 0 0 0 1 48" "80 0 0 0 1 32" "80 0 0 0 1 40" "80 0 0 0 1 -16" "80 0 0 0 1 44" "80 0 0 0 1 42" ; do timeout 20 tools/probes/tma_probe $args 2>&1 | tail -1; done
