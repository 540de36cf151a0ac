# A/B library variants: scratch/ab_build.sh NAME "-DFLAG=..." -> paper_2505_15909_b200/librtnq_b200_NAME.so
name=$1; flags=$2
RTNQ_EXTRA_CUFLAGS="$flags" python -c "
import sys; sys.path.insert(0,'.')
import paper_2505_15909_b200.build as b
b.OBJ = b.OBJ + '_$name'; b.LIB = b.LIB.replace('librtnq_b200.so','librtnq_b200_$name.so'); b.build()" 2>&1 | grep -i error
