# build _variants/$1.so with the -D flags in $2; only csrc unit $3 (e.g. fmp_omp_c64.cu) is recompiled
set -e
name=$1; defs=$2; unit=$3
obj=_variants/${name}_obj
mkdir -p $obj
cp paper_1205_4139_b200/_build/*.o $obj/
rm -f $obj/$unit.o
touch $obj/*.o
FMP_BUILD_DEFS="$defs" FMP_BUILD_OUT=_variants/$name python -m paper_1205_4139_b200.build
rm -rf $obj
echo built $name
