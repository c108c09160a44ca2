for v in A B C D E A B C D E; do python tools/variant_apply.py tools/var/lib_$v.so cfg4 4; done
