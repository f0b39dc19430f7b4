cd $GRAFT_REPO_ROOT
GRASS_LIB_PATH=$GRAFT_REPO_ROOT/build/mutants/libgrass_m12.so timeout 300 python tools/dbg_m12.py > gpurun_out/r14_m12.log 2>&1
timeout 300 python tools/dbg_m12.py >> gpurun_out/r14_m12.log 2>&1
