timeout 60 ./tools/micro/pipe3
