#!/bin/bash
# Final round-2 refresh (one box, one call): every bench line (full-size parity leg, threaded
# oracle baseline), then the ncu evidence of profiles/tools/ncu_r02.sh for the Higgs line.
bash profiles/tools/refresh_r02.sh
bash profiles/tools/ncu_r02.sh
echo refresh_done
