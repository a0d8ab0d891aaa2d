/*
 * levyh_b200_testing.h -- test and diagnostic hooks of liblevyh_b200_testing.so (not part of
 * the drop-in ABI in levyh_b200.h): plan export for the CPU plan emulator
 * (tests/plan_emulator.py), planner timing, and executor / recompression micro-benchmarks.
 * The testing library links against liblevyh_b200.so.
 */
#ifndef LEVYH_B200_TESTING_H
#define LEVYH_B200_TESTING_H

#include "levyh_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Host-only: write the block layouts and the H-LU / solve / inverse task DAGs of this
 * partition to `path` (binary, see tests/plan_emulator.py) for CPU verification. */
int lh_debug_dump_plans(const lh_tree *rt, const lh_tree *ct, int n_min, int n_block, double eta,
                        int kcap_f, int kcap_x, const char *path);
/* Host-only planner timing on the partition of (rt, ct): which & 1 plans the H-LU, which & 2
 * the propagator; out[0..3] = H-LU plan seconds, tasks, propagator plan seconds, tasks. */
int lh_debug_plan_timing(const lh_tree *rt, const lh_tree *ct, int n_min, int n_block, double eta,
                         int kcap_f, int kcap_x, int which, double *out);
/* Executor micro-benchmark: R synthetic tasks of one kind (0 GETRF 64x64 + leaf inverse,
 * 1 TRSM via leaf inverse, 2 SEGMUL with one dense 64x64 piece), k right-hand columns,
 * chained (each depends on the previous) or independent.  out[0] = wall us per task,
 * out[1] = mean task body us (device timestamps). */
int lh_debug_task_bench(lh_ctx *ctx, int kind, int R, int k, int chain, double *out_host);
/* Debug: phase-timed recompression (QR(U), QR(V), Ru Rv^T, Jacobi SVD, truncation + apply) of
 * host U (m x K), V (n x K) on every SM, reps times; out[0..5] mean ns per phase, out[6] rank.
 * Times the kernel behind hops.py:134-144 (_lowrank_add_recompress). */
int lh_debug_recomp_bench(lh_ctx *ctx, int m, int n, int K, int reps, const double *u_host,
                          const double *v_host, double *out_host);

#ifdef __cplusplus
}
#endif

#endif
