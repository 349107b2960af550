python -m paper_2005_06727_b200.build > /dev/null 2>&1
for c in tweet scaling; do
 echo "== k16s3 $c"; python tools/pass_timing.py $c auto 5
 for v in k8 k8s4 k32; do echo "== $v $c"; WMD_LIB=variants/lib_$v.so python tools/pass_timing.py $c auto 5; done
done
