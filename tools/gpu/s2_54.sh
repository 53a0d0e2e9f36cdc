cd tools/micro; timeout 120 ./dec_copies 2>&1 | tail -12
