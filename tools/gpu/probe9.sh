timeout 60 ./tools/micro/mbar_cost
