bash tools/full_check.sh
TAG=r01h CONFIGS="2 3 4 5" bash tools/ncu_round.sh
