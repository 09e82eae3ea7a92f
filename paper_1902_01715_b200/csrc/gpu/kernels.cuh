// Device data layout + kernel launchers for the sm_100a solve path.
//
// Everything is fp64 on CUDA cores: the path is sparse and HBM-bound
// ("None use tensor cores"). Indices are int32 on the device
// (all configs have nnz < 2^31), which cuts index traffic vs the reference's
// int64 CSR (sparse_matrix.hpp:27-33).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace aspamg_gpu {

constexpr int kBlock = 256;  // threads per CTA for every streaming kernel

// CSR, int32 offsets/columns. `group` = threads cooperating on one row
// (power of two, 1..256), chosen from the row lengths at upload.
struct DCsr {
    int n_rows = 0, n_cols = 0;
    long long nnz = 0;
    int* rp = nullptr;
    int* ci = nullptr;
    double* v = nullptr;
    int group = 1;
    int pol = 0;  // L2 policy of the matrix stream: 0 default, 1 evict-first, 2 evict-last
    // 16-bit column offsets (instead of ci) when every row's columns span < 2^16:
    // column = cb[row] + ci16[k] (10 instead of 12 matrix bytes per entry)
    unsigned short* ci16 = nullptr;
    int* cb = nullptr;
    int pf = 0;  // k_csr row-pointer prefetch (T <= 16)
    int blk = 0; // k_csrw: 1 = contiguous row block per CTA (L1 reuse of x across steps), 0 = rows interleaved over the grid
    int wu = 0;  // > 0: warp-per-row pipelined kernel k_csrw (group == 32, 32-bit columns), wu columns per lane per round
    // Long-row split: rows longer than lthr (listed in lrows) are computed by the
    // first nlctas CTAs of the launch, one warp per row; the regular T-thread
    // groups skip them, so a long-tailed operand (G' rows up to ~7x the mean) no
    // longer waits on a few long serial chains.
    int nlong = 0, lthr = 0, nlctas = 0;
    int* lrows = nullptr;
};

// Sliced 3x3-block format for an exactly 3x3-blocked operator (K): block
// rows are grouped in chunks of 32, one lane per block row. Chunk c has
// width[c] block slots (the longest block row of the chunk) starting at slot
// off[c]; slot j of lane l holds block column ci[(off+j)*32 + l] and the
// block's 9 values (row-major) at v[((off+j)*9 + e)*32 + l]. Every warp load
// is a contiguous 256-B (values) / 128-B (columns) line; each lane sums its
// three rows sequentially in ascending column order (the reference's order,
// sparse_matrix.cpp:100-105). Block rows shorter than the chunk width are
// padded; padded slots are predicated off (never loaded).
struct DSbsr3 {
    int nb = 0, nbc = 0, nchunks = 0;
    long long nnzb = 0, slots = 0;  // slots = padded block slots (incl. padding), per lane x 32
    int* len = nullptr;             // blocks per block row
    int2* meta = nullptr;           // per chunk {off, width}
    int* ci = nullptr;
    double* v = nullptr;
    int pol = 0;
};

// SELL-32 (sliced ELL, chunk height 32, no sorting): one lane per row,
// same slot-major layout as DSbsr3 with scalar entries. Used for short rows
// (G, G', P, P', short coarse A_l): coalesced, no cross-lane reduction,
// sequential ascending-column sums.
struct DSell {
    int n_rows = 0, n_cols = 0, nchunks = 0;
    long long nnz = 0, slots = 0;
    int chh = 32;         // chunk height: 32 (one chunk per warp) or 8 (four chunks per warp)
    int* perm = nullptr;  // SELL-32-sigma: slot row -> matrix row (null = natural order)
    int* len = nullptr;   // per slot row
    int u = 81;           // register-pipelined variant: U*10 + min CTAs/SM (81, 83, 84, 41, 44, 46, 21)
    int2* meta = nullptr;
    int* ci = nullptr;
    double* v = nullptr;
    int pol = 0;
    unsigned short* ci16 = nullptr;  // 16-bit column offsets: column = cb[slot row] + ci16[slot]
    int* cb = nullptr;
};

// Tile-local SELL ("xsell"): rows in tiles of R rows (one CTA of R threads per
// tile, one lane per row). Per tile the kernel first stages the tile's x
// FOOTPRINT — the sorted list of the 2^gran-double granules of x its entries
// reference — into shared memory with 16-B cp.async copies (each granule read
// once per tile, fully coalesced), and the matrix stores 16-bit LOCAL columns
// (granule rank << gran | offset) into that staged window. The x gathers of the
// row sums then hit shared memory (bank conflicts only) instead of costing one
// L1 wavefront per distinct line per warp instruction, which is what bounds
// the lane-per-row kernels on scattered columns. Inside a tile the rows are
// sorted by length (descending, stable) so each 32-row chunk is nearly
// rectangular (with fold = 2 a lane owns two rows, rank t and rank R-1-t, whose
// quads follow each other in the chunk); slots are stored in groups of four per lane ("quads": one 8-B
// load of four 16-bit columns, two 16-B loads of values), chunk widths padded
// to whole quads, padded entries predicated off. Local columns keep the
// ascending global order, and every lane sums its row sequentially with
// separate multiply / add: y is bit-identical to the reference spmv
// (sparse_matrix.cpp:100-105).
struct DXsell {
    int n_rows = 0, n_cols = 0, ntiles = 0;
    int R = 256;     // tile height (rows); the CTA has R / fold threads
    int fold = 1;    // rows per lane: 1, or 2 = sorted rank t paired with rank R-1-t (balances the warps)
    int gran = 3;    // log2 doubles per footprint granule
    long long nnz = 0, quads = 0, list_len = 0;
    int2* tmeta = nullptr;           // per tile {list offset, granule count}
    int2* cmeta = nullptr;           // per chunk {quad offset, width of the a rows | width of the b rows << 16}
    unsigned short* len = nullptr;   // per slot row (sorted order), padded to ntiles * R
    unsigned short* perm = nullptr;  // per slot row: local row inside the tile
    int* list = nullptr;             // footprint granule ids, tile after tile
    double2* v = nullptr;            // quad q of a chunk, half h, lane l at v[((off + q) * 2 + h) * 32 + l]
    uint2* lc = nullptr;             // quad q, lane l at lc[(off + q) * 32 + l]: four 16-bit local columns
    int fp_doubles = 0;              // staged window capacity (largest tile footprint), in doubles
    int pol = 0;
    int q = 2;                       // quads per load group (kernel variant)
};

// One matrix operand.
struct DMat {
    int fmt = 0;  // 0 CSR (group per row), 1 sliced BSR3, 2 SELL-32, 3 tile-local SELL
    DCsr csr;
    DSbsr3 sb;
    DSell sell;
    DXsell xs;
    int rows() const { return fmt == 1 ? 3 * sb.nb : fmt == 2 ? sell.n_rows : fmt == 3 ? xs.n_rows : csr.n_rows; }
    int cols() const { return fmt == 1 ? 3 * sb.nbc : fmt == 2 ? sell.n_cols : fmt == 3 ? xs.n_cols : csr.n_cols; }
    long long nnz() const { return fmt == 1 ? 9 * sb.nnzb : fmt == 2 ? sell.nnz : fmt == 3 ? xs.nnz : csr.nnz; }
};

// Epilogue of y = f(M x):
enum Epi : int {
    EPI_PLAIN = 0,     // y = Mx
    EPI_SCALE = 1,     // y = omega * Mx
    EPI_RESID = 2,     // y = aux - Mx
    EPI_ADD = 3,       // y = aux + Mx
    EPI_ADDSCALE = 4,  // y = aux + omega * Mx
};

// What the last CTA does with a finished deterministic reduction.
enum Fin : int {
    FIN_NONE = 0,
    FIN_STORE = 1,   // out[0] = sum
    FIN_PQ = 2,      // PCG: pq = sum; alpha = rz/pq; pq <= 0 -> not SPD, done
    FIN_RZ = 3,      // PCG: beta = (k == 0) ? 0 : sum/rz ; rz = sum
    FIN_RR = 4,      // PCG: history[k] = sqrt(sum)/||b||; k++; convergence test
    FIN_INIT = 5,    // PCG init (two sums: b.b, r.r)
};

// Device-resident PCG state (one per context). Host reads it once per solve.
struct PcgState {
    double rz, pq, alpha, beta, bnorm, tol, rr, trr2;
    long long k, max_it;
    int done, notspd, converged, pad;
    double* history;
};

// Deterministic two-pass reduction site: every CTA writes its fixed-order
// partial, the last CTA to arrive (atomic ticket) sums the partials in index
// order -> same bits for every run, no floating-point atomics.
struct Red {
    double* partials = nullptr;   // >= gridDim.x (x2 for FIN_INIT)
    unsigned* counter = nullptr;
    int fin = FIN_NONE;
    double* out = nullptr;
    PcgState* st = nullptr;
    unsigned long long cond = 0;  // cudaGraphConditionalHandle for FIN_RR (0 = none)
    int use_cond = 0;
};

struct Launch {
    int grid = 0;
    cudaStream_t stream = nullptr;
};

// y = epi(M x); optional dot sum_i y_i * dotw_i reduced through `red`.
// `done` (device int) makes the kernel a no-op once the solve has finished.
void spmv(const DMat& M, Epi epi, const double* x, double* y, const double* aux, double omega,
          const double* dotw, const Red& red, const int* done, const Launch& L);
int spmv_grid(const DMat& M);

// p = (k == 0) ? z : z + beta p
void pcg_p(int n, const double* z, double* p, const PcgState* st, const int* done, const Launch& L);
// x += alpha p ; r -= alpha q ; rr = r.r -> FIN_RR
void pcg_xr(int n, double* x, double* r, const double* p, const double* q, const Red& red, const int* done,
            const Launch& L);
// b.b and r.r -> FIN_INIT
void pcg_init_dots(int n, const double* b, const double* r, const Red& red, const Launch& L);
int vec_grid(int n);

// Coarsest level, "forward and backward solve" L L' z = y.
// mode 0: blocked substitution in one CTA (Lrm row-major L, Lcm row-major L',
//         Dinv_f / Dinv_b inverted 32x32 diagonal blocks).
// mode 1: the two triangular solves applied through the explicit inverse
//         factor W = L^{-1} (computed once at upload): w = W y, z = W' w, each a
//         multi-CTA CSR product over the dense triangle (context.cu).
void coarse_solve(int n, const double* Lrm, const double* Lcm, const double* Dinv_f, const double* Dinv_b,
                  const double* y, double* z, const double* dotw, const Red& red, const int* done, const Launch& L);

// ------------------------------------------------------------ coarse tail
// The small levels of the V-cycle run as ONE persistent kernel that walks a
// device-side op table (CSR products with epilogues, zero fills) with a
// software grid barrier between ops: the ~20 launches / drains of the tail
// become one launch; all CTAs are co-resident (cooperative launch).
struct TailOp {
    int kind;  // 0 CSR product, 1 zero fill
    int epi;
    DCsr M;
    const double* x;
    double* y;
    const double* aux;
    double omega;
    int n;     // rows for kind 1
};
struct GridBar {
    unsigned count;
    unsigned gen;
};
void tail_run(const TailOp* ops, int nops, GridBar* bar, const int* done, int grid, cudaStream_t s);
int tail_grid();
// r = y - A s (sliced BSR3) and r_c = P' r (pt: a CSR product op, x = r) in one
// cooperative launch with a grid barrier in between (option "fuse_rr").
void resid_restrict(const DSbsr3& A, const TailOp& pt, const double* s, double* r, const double* y, GridBar* bar,
                    const int* done, int grid, cudaStream_t st);
int resid_restrict_grid(int pol);

void set_pdl(bool on);          // programmatic dependent launch on/off (process-wide)
void spmv_prepare();          // once per process, outside any stream capture
void xsell_prepare(const DXsell& M);  // once per operand, outside any stream capture (dynamic smem opt-in)
void coarse_prepare(int n);  // once per factor size, outside any stream capture
void fill_zero(int n, double* y, const int* done, const Launch& L);

}  // namespace aspamg_gpu
