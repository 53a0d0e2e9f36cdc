timeout 60 ./tools/micro/mma_acc
