#!/bin/bash
# Round-end measurement run (one B200, under gpurun): bench lines, ncu launch list, ncu full captures of the hot
# kernels (summarised here; the .ncu-rep files stay in /tmp on the box), executed FP64 flops per config, parity
# report, LU sweep.  Text outputs go to gpurun_out/f_*.
P=/tmp/podp_prof; mkdir -p $P gpurun_out
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-adapt > gpurun_out/f_launch_run.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:'lu_ll|mpt_tile' -c 2 -o $P/c2_full python tools/prof_run.py 2 1 > gpurun_out/f_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
python tools/ncu_summary.py $P/c2_full.ncu-rep > gpurun_out/f_ncu_full_c2_F1e5.txt 2>&1
python tools/ncu_phase.py $P/c2_full.ncu-rep paper_2307_05590_b200/build/k_lu_ll.cu.o lu_ll_kernelILi48ELb1ELb0ELb1ELb0 regex:lu_ll > gpurun_out/f_ncu_phase_ll48.txt 2>&1
ncu -i $P/c2_full.ncu-rep --page raw --csv > $P/c2_raw.csv
python - <<'PY' > gpurun_out/f_ncu_metrics_c2.txt
import csv
rows = list(csv.reader(open('/tmp/podp_prof/c2_raw.csv')))
h, u = rows[0], rows[1]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__icc_request_hit_rate.pct', 'gcc__cache_requests_type_instruction.sum.pct_of_peak_sustained_elapsed',
        'smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'sm__warps_active.avg.per_cycle_active', 'smsp__inst_executed.sum']
for d in rows[2:]:
    m = dict(zip(h, d)); uu = dict(zip(h, u))
    print('==', m.get('Kernel Name'))
    for k in keys:
        print(f'  {k:86s} {m.get(k)} {uu.get(k)}')
PY
ncu --set full --clock-control none --import-source on -k regex:'lu_ll' -c 1 -o $P/c4_full python tools/prof_run.py 4 1 20000 > gpurun_out/f_ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
python tools/ncu_summary.py $P/c4_full.ncu-rep > gpurun_out/f_ncu_full_c4_ll96_F20000.txt 2>&1
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for c in 0 1 2 3 4; do F=""; [ $c = 4 ] && F=100000; ncu --metrics $M --clock-control none -k regex:'lu_ll|mpt_tile' -c 2 --csv --log-file $P/flops_c$c.csv python tools/prof_run.py $c 1 $F > /dev/null 2>&1; done
python tools/flops_summary.py $P/flops_c0.csv $P/flops_c1.csv $P/flops_c2.csv $P/flops_c3.csv $P/flops_c4.csv > gpurun_out/f_executed_flops_by_config.txt 2>&1
python tools/parity_report.py > gpurun_out/f_parity.jsonl 2> gpurun_out/f_parity.err; echo "parity rc=$?"
python tools/lu_ab.py 8 16 24 32 40 48 56 64 72 80 88 96 > gpurun_out/f_lu_sweep.txt 2>&1
python tools/mpt_ab.py > gpurun_out/f_mpt_ab.txt 2>&1
du -sh gpurun_out
