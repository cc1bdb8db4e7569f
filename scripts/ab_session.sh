o=gpurun_out/checked; mkdir -p $o
NSL_LIB=$PWD/abl/libnsl_checked.so timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $o/tests.log 2>&1; echo rc=$? >> $o/tests.log
