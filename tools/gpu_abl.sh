#!/bin/bash
for t in qrp qrpDCORU_ABL_NO_TRAIL qrpDCORU_ABL_CHAIN_ONLY; do echo "== $t"; timeout -s KILL 60 ./tools/$t 4000 60 | head -2; timeout -s KILL 60 ./tools/$t 960 60 | head -2; done
