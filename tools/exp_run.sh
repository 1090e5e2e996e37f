cp exp/libkfbi_exp2.so paper_2404_15249_b200/lib/libkfbi.so; touch paper_2404_15249_b200/lib/libkfbi.so; bash tools/ncu_kd.sh C3 "k_inv_sparse" 0 expinv2
