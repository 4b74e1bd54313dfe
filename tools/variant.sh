# build a variant library from the current sources: bash tools/variant.sh NAME  -> variants/libiga_NAME.so
set -e
mkdir -p variants
NAME=$1
python -c "
import paper_1305_4452_b200.build as b, os, shutil
b.BUILD = os.path.join(b.HERE, 'build_var'); b.SO = os.path.join(os.getcwd(), 'variants', 'libiga_$NAME.so')
b.build()
"
echo variants/libiga_$NAME.so
