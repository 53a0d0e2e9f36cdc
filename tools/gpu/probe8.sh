timeout 120 ./tools/micro/stream2
