bash exp/ab_libs.sh build/ab/oldcl.so build/ab/v8.so
bash exp/ab_libs.sh build/ab/oldcl.so build/ab/v8.so
