bash tools/ab.sh DINFER_K34_LATE 0 1 3
bash tools/ab.sh DINFER_K34_FLAGS 0 1 2
