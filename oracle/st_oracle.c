/*
 * ORACLE — plain, slow, obviously-correct CPU implementation of the
 * SCALE-TRACK two-way-coupled Lagrangian particle step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2603_26691_b200/) never imports, links or calls it, and
 * shares no code, header or constant with it.
 *
 * What it follows (PAPER.md = P, SPEC.md = S, readings C-n in DESIGN.md §3):
 *   - Newton's law for a particle, Eq. 9-10, drag only plus an
 *     optional body acceleration (C-1), Schiller-Naumann factor (C-2),
 *     tau_p = rho_p d^2/(18 rho_f nu_f) (C-3), exponential (C-4) or
 *     semi-implicit Euler integration over a fixed sub-step;
 *   - momentum source Eq. 11, deposited into the cell containing
 *     the particle at the sub-step start (C-10), fluid-side sign (C-8);
 *   - reflecting walls or periodic wrap (C-12);
 *   - cell location floor((x - o)/h) with upper boundary -> last cell (C-6).
 *   - stable counting sort by chunk id for the rebin (C-15).
 * Parity pins: tests/test_oracle_pins.py (P-1 .. P-11 of DESIGN.md §5).
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared (see Makefile).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_BC_PERIODIC = 0, ORC_BC_REFLECT = 1 };
enum { ORC_DRAG_STOKES = 0, ORC_DRAG_SCHILLER_NAUMANN = 1 };
enum { ORC_INT_EXPONENTIAL = 0, ORC_INT_SEMI_IMPLICIT = 1 };
enum { ORC_ONE_WAY = 0, ORC_TWO_WAY = 1 };
enum { ORC_OK = 0, ORC_ERR_CFL = 5 };

/* The oracle's own parameter block (mirrored by oracle/__init__.py). */
typedef struct {
  int32_t dims[3];
  double origin[3];
  double cell_size[3];
  int32_t chunk_cells;
  int32_t bc[3];
  double rho_f, nu_f, rho_p;
  double gravity[3];
  int32_t drag_law, integrator, coupling;
} orc_params;

/* ---- fp32-state mode: every operation rounded to binary32 ---- */
#define REAL float
#define SFX(name) name##_f32
#define FLOOR floorf
#define SQRT sqrtf
#define EXP expf
#define EXPM1 expm1f
#define POW powf
#include "st_oracle_step.inc"
#undef REAL
#undef SFX
#undef FLOOR
#undef SQRT
#undef EXP
#undef EXPM1
#undef POW

/* ---- fp64 mode: closed-form and conservation pins ---- */
#define REAL double
#define SFX(name) name##_f64
#define FLOOR floor
#define SQRT sqrt
#define EXP exp
#define EXPM1 expm1
#define POW pow
#include "st_oracle_step.inc"
#undef REAL
#undef SFX
#undef FLOOR
#undef SQRT
#undef EXP
#undef EXPM1
#undef POW

/*
 * C-15: stable counting sort of n items by key in [0, nkeys) (the bin key of
 * orc_bin_key_*, or any integer key).  perm receives
 * the store order after the sort (perm[j] = old index of the item now at j);
 * offsets (nkeys+1 entries, may be NULL) receives the CSR bin offsets.
 * Returns -1 on a key out of range.
 */
int orc_stable_order(int64_t n, const int64_t* key, int64_t nkeys, int64_t* perm,
                     int64_t* offsets) {
  int64_t* start = (int64_t*)calloc((size_t)nkeys + 1, sizeof(int64_t));
  if (!start) return -2;
  for (int64_t i = 0; i < n; ++i) {
    if (key[i] < 0 || key[i] >= nkeys) { free(start); return -1; }
    start[key[i] + 1] += 1;                       /* count */
  }
  for (int64_t k = 0; k < nkeys; ++k) start[k + 1] += start[k];   /* exclusive prefix */
  if (offsets) memcpy(offsets, start, ((size_t)nkeys + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) perm[start[key[i]]++] = i;     /* place in input order */
  free(start);
  return 0;
}

int orc_abi(void) { return 1; }
