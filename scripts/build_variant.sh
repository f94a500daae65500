# build a variant of the library with extra nvcc flags: build_variant.sh NAME "-DFOO=1 ..."
# -> paper_2104_06784_b200/libtpflow_b200_NAME.so (development A/B aid)
set -e
cd "$(dirname "$0")/.."
make -s -C paper_2104_06784_b200/csrc OUT=$PWD/paper_2104_06784_b200/libtpflow_b200_$1.so \
    OBJ=$PWD/paper_2104_06784_b200/csrc/build_$1 EXTRA="$2" $PWD/paper_2104_06784_b200/libtpflow_b200_$1.so > /dev/null
grep -A2 "stage_kernelILb1ELb[01]" paper_2104_06784_b200/csrc/build_$1/ptxas.log | grep spill | tr '\n' ' '; echo
