for v in A B C D A B C D; do python tools/variant_apply.py tools/var/lib_$v.so cfg4 4; done
