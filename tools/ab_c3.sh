for lib in lut lut_el line_ef both; do echo "=== $lib"; FMG_LIB_PATH=tools/ab/$lib.so python tools/prof_c3.py 1000000 4 2>&1 | tail -2; done
echo "=== lut K13"; FMG_LUT_K=13 python tools/prof_c3.py 1000000 4 2>&1 | tail -2
echo "=== lut_el K13"; FMG_LUT_K=13 FMG_LIB_PATH=tools/ab/lut_el.so python tools/prof_c3.py 1000000 4 2>&1 | tail -2
