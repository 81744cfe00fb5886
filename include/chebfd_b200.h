/*
 * chebfd_b200.h -- C ABI of the B200-native Chebyshev filter diagonalization
 * hot path (libchebfd_b200.so).  Plain pointers and sizes only; complex
 * numbers are interleaved (re, im) float64 pairs; block-vector panels keep the
 * reference layout, element (i, j) of a width-nb panel at i*ld + j
 * (reference: proj/include/chebfilter/block_vector.hpp:49-52, 81-94).
 *
 * Every entry returns 0 on success or a CF_E* code mapped 1:1 to the
 * reference's exception types (std::invalid_argument, std::out_of_range,
 * std::runtime_error, ProtocolError); cf_last_error() returns the message of
 * the calling thread's last failure.  There is no CPU fallback: device entry
 * points fail with CF_ECUDA when no sm_100 device is usable.
 *
 * Each declaration cites the reference interface it replaces (file:line,
 * relative to the reference repo root).
 */
#ifndef CHEBFD_B200_H
#define CHEBFD_B200_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define CF_OK 0
#define CF_EINVAL 1    /* std::invalid_argument */
#define CF_ERANGE 2    /* std::out_of_range */
#define CF_ERUNTIME 3  /* std::runtime_error */
#define CF_EPROTOCOL 4 /* chebfilter::ProtocolError (dist.hpp:102-104) */
#define CF_ECUDA 5     /* CUDA failure / no usable device */

const char* cf_last_error(void);
int cf_version(void);

/* ------------------------------------------------ host-side routines ---- */
/* topi_generate (sparse_matrix.hpp:181-228): closed-form row generator,
 * bit-identical CRS.  Two-phase: row_ptr == NULL returns n and nnz only. */
int cf_topi_generate(size_t nx, size_t ny, size_t nz, double mass, double hop, int open_boundary, size_t* n,
                     size_t* nnz, uint64_t* row_ptr, int32_t* col_idx, double* values);
/* gershgorin_bounds (sparse_matrix.hpp:89-107) */
int cf_gershgorin_bounds(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, double* lo,
                         double* hi);
/* spectral_map (filter.hpp:25-32) */
int cf_spectral_map(double lambda_min, double lambda_max, double margin, double* alpha, double* beta);
/* filter_coefficients (filter.hpp:39-70); damping 0 = jackson, 1 = none; c, g: np+1 */
int cf_filter_coefficients(double window_lo, double window_hi, double alpha, double beta, size_t np, int damping,
                           double* c, double* g);
/* BlockVector(n, n_s, n_b, InitSeededRandom{seed, row_offset}) (block_vector.hpp:57-73):
 * panel-concatenated output, n_s/n_b panels of n*n_b complex. */
int cf_blockvec_random(size_t n, size_t ns, size_t nb, uint64_t seed, uint64_t row_offset, double* out);
/* The same vector generated on the device into npanels = ns/nb device panels
 * (columns j0..ns-1 only), for block vectors too large for the host: integer
 * hashes bit-identical, Box-Muller values within 1-2 ulp of the host's libm. */
int cf_blockvec_random_device(size_t n, size_t ns, size_t nb, uint64_t seed, uint64_t row_offset, void* const* panels,
                              size_t j0, void* stream);
/* partition_rows (partition.hpp:28-60).  ranges: 2*workers.  halo_in flattened
 * as records (w, v, count, rows...) for w, v ascending; halo == NULL sizes it. */
int cf_partition_rows(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, size_t workers, uint64_t* ranges,
                      uint64_t* halo, size_t* halo_len);
/* shard_and_distribute (dist.hpp:39-98) for worker w: local CRS with remapped
 * columns, halo_global, send/recv plans flattened as (neighbor, count, rows...).
 * Two-phase: rp == NULL returns the sizes only. */
int cf_shard(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const double* values, size_t workers, size_t w,
             size_t* row_begin, size_t* local_n, size_t* halo_n, size_t* nnz, uint64_t* rp, int32_t* ci, double* v,
             uint64_t* halo_global, uint64_t* send_flat, size_t* send_len, uint64_t* recv_flat, size_t* recv_len);

/* Shard w of a Topi lattice partitioned over `workers` (partition_rows +
 * shard_and_distribute, dist.hpp:39-98, applied to topi_generate) generated in
 * closed form from the worker's own rows, without building the global matrix.
 * Send plans use the symmetric sparsity pattern of the Hermitian stencil.
 * Same outputs and two-phase protocol as cf_shard. */
int cf_topi_shard(size_t nx, size_t ny, size_t nz, double mass, double hop, int open_boundary, size_t workers,
                  size_t w, size_t* row_begin, size_t* local_n, size_t* halo_n, size_t* nnz, uint64_t* rp, int32_t* ci,
                  double* v, uint64_t* halo_global, uint64_t* send_flat, size_t* send_len, uint64_t* recv_flat,
                  size_t* recv_len);

/* ---------------------------- SELL-C-sigma over 4x4 blocks (new format) ---
 * The reference stores CRS only (sparse_matrix.hpp:22-33; SELL-C-sigma is a
 * SPEC non-goal).  The device format groups rows into 4-row block-rows and
 * columns into 4-column block-columns; each block keeps a 16-bit pattern mask
 * and its nonzeros packed row-major, so every U block-column is gathered once
 * per block-row.  Block-rows are taken in `order` (a locality schedule; NULL =
 * natural), stable-sorted by descending block count inside windows of `sigma`
 * block-rows, and cut into chunks of C block-rows.  perm[slot] = block-row. */
int cf_sell_permutation(size_t n, const uint64_t* row_ptr, const int32_t* col_idx, const int32_t* order, int C,
                        int sigma, int32_t* perm_out, size_t* nslots);
/* Host-side SELL-C-sigma/B4 build statistics (no device needed): stats[9] =
 * {chunks, piece records, work units, staged (every chunk has a plan),
 * signature chunks, max runs per plan, max staged block columns per chunk,
 * total staged block columns, record bytes}. */
int cf_sell_layout_stats(size_t n, size_t ncols, const uint64_t* row_ptr, const int32_t* col_idx,
                         const double* values, const int32_t* order, size_t* stats);
/* Locality schedule for a lattice matrix (rows = 4*((z*ny+y)*nx+x)+r): xy tiles
 * of tx*ty sites marched along z.  Writes nx*ny*nz block-row ids. */
int cf_lattice_order(size_t nx, size_t ny, size_t nz, size_t tx, size_t ty, int32_t* order);
/* The same with the planes z = 0 and z = nz-1 first (a z-slab shard's boundary planes:
 * its halo reads and halo sends happen in the first work units of a step). */
int cf_lattice_order_boundary_first(size_t nx, size_t ny, size_t nz, size_t tx, size_t ty, int32_t* order);

/* ------------------------------------------------------------ file I/O ---
 * matrix_market_read (matrix_market.hpp:22-81): "matrix coordinate complex"
 * general or hermitian (lower triangle, expanded), duplicates summed in file
 * order as build_from_triplets.  Two-phase: row_ptr == NULL parses and returns
 * n, nnz and symmetry (0 hermitian, 1 general); the next call with buffers for
 * the same path copies the parsed matrix.  Parse errors return CF_ERUNTIME and
 * cf_matrix_market_error_line() gives MatrixMarketError::line_number. */
int cf_matrix_market_read(const char* path, size_t* n, size_t* nnz, int* symmetry, uint64_t* row_ptr,
                          int32_t* col_idx, double* values);
size_t cf_matrix_market_error_line(void);
/* matrix_market_write (matrix_market.hpp:85-104): byte-identical output. */
int cf_matrix_market_write(const char* path, size_t n, const uint64_t* row_ptr, const int32_t* col_idx,
                           const double* values, int symmetry);
/* block_vector_write / block_vector_read (block_vector.hpp:182-229), CFDB v1;
 * panels: host, panel-concatenated n_s/n_b panels of n x n_b complex.
 * Read is two-phase: panels == NULL returns the shape. */
int cf_blockvec_write(const char* path, size_t n, size_t ns, size_t nb, const double* panels);
int cf_blockvec_read(const char* path, size_t* n, size_t* ns, size_t* nb, double* panels);

/* ------------------------------------------------------ device matrix --- */
/* Block vectors (block_vector.hpp:53-151): rows x n_s complex as n_s/n_b device
 * panels, each row-major rows x n_b (the reference's panel layout); created
 * zeroed (InitZero).  upload / download move all panels, panel-concatenated
 * (n_s/n_b, rows, n_b) like BlockVector's storage.  cf_panel_swap is
 * swap_blocks (block_vector.hpp:138-146): exchanges the two panel buffers, O(1);
 * shape mismatch -> CF_EINVAL, panel index -> CF_ERANGE. */
typedef struct cf_blockvec_s* cf_blockvec;
int cf_blockvec_create(int device, size_t rows, size_t ns, size_t nb, cf_blockvec* out);
int cf_blockvec_destroy(cf_blockvec v);
int cf_blockvec_shape(cf_blockvec v, size_t* rows, size_t* ns, size_t* nb, int* device);
int cf_blockvec_panel(cf_blockvec v, size_t b, void** dev_ptr);
int cf_blockvec_upload(cf_blockvec v, const double* host_panels);
int cf_blockvec_download(cf_blockvec v, double* host_panels);
int cf_panel_swap(cf_blockvec a, size_t ia, cf_blockvec b, size_t ib);

typedef struct cf_matrix_s* cf_matrix;
/* Build (host, threaded) and upload.  ncols >= n: columns >= n address halo
 * rows of the block vectors (dist.hpp:19-37).  C = 0, sigma = 0 pick defaults. */
int cf_matrix_create_crs(int device, size_t n, size_t ncols, const uint64_t* row_ptr, const int32_t* col_idx,
                         const double* values, const int32_t* order, int C, int sigma, cf_matrix* out);
/* topi_generate + build in one step with the lattice locality schedule. */
int cf_matrix_create_topi(int device, size_t nx, size_t ny, size_t nz, double mass, double hop, int open_boundary,
                          cf_matrix* out);
/* Device matrix of worker w's shard of a Topi lattice over `workers` row blocks
 * (partition_rows + shard_and_distribute, dist.hpp:39-98, generated in closed
 * form as cf_topi_shard): local_n rows, local_n + halo_n columns; whole-plane
 * slabs keep the lattice locality schedule.  The rank-local operator of a
 * multi-GPU run, without a host copy of the global matrix. */
int cf_matrix_create_topi_shard(int device, size_t nx, size_t ny, size_t nz, double mass, double hop,
                                int open_boundary, size_t workers, size_t w, size_t* row_begin, size_t* local_n,
                                size_t* halo_n, cf_matrix* out);
int cf_matrix_info(cf_matrix m, size_t* n, size_t* ncols, size_t* nnz, size_t* device_bytes, size_t* units);
/* 1 when every chunk has a staging plan (n_b = 32 panels run the chunk-staged TMA kernel). */
int cf_matrix_staged(cf_matrix m, int* staged);
/* 1 when whole-row n_b = 2 / 4 / 8 / 12 / 16 panels of this matrix run the narrow chunk-staged
 * kernel (every chunk one typed record with a staging plan; knobs "staged",
 * "typed" and "narrow" on), else the register-gather kernel.  Introspection only. */
int cf_matrix_narrow(cf_matrix m, int* narrow);
/* Pieces stored as typed records (purely real / imaginary values, one double
 * each) out of all pieces; a matrix mixes typed and full records per piece. */
int cf_matrix_typed(cf_matrix m, size_t* typed_pieces, size_t* pieces);
/* Declare rows [0, rows_lo) and [n - rows_hi, n) the shard's boundary rows (they read
 * halo columns or are mirrored to neighbours); *units = the leading work units that
 * hold them (0: none).  cf_matrix_create_topi_shard sets it for its slabs. */
int cf_matrix_set_boundary(cf_matrix m, size_t rows_lo, size_t rows_hi, int* units);
/* Export the stored matrix back to CRS (round-trip check); two-phase like cf_topi_generate. */
int cf_matrix_to_crs(cf_matrix m, size_t* n, size_t* nnz, uint64_t* row_ptr, int32_t* col_idx, double* values);
int cf_matrix_destroy(cf_matrix m);

/* ------------------------------------------------------ device memory ---
 * Plain device allocations and copies for callers that do not link the CUDA
 * runtime themselves (include/chebfilter_b200.hpp keeps its panels here).
 * kind: 0 host->device, 1 device->host, 2 device->device.  Synchronous. */
int cf_device_count(int* count);
/* Kernel-variant knobs for A/B runs (process-wide; unknown key -> CF_EINVAL):
 *   "staged"  1 (default) chunk-staged TMA kernel where a matrix has staging
 *             plans, 0 register-gather kernel;
 *   "x_group" degrees per X update in apply_filter: 3 (default), 2, 1 (every
 *             step, the reference's schedule);
 *   "wpf"     producer L2 prefetch of epilogue rows: pieces ahead in the low 4
 *             bits, +16 = X rows too (default 18), 0 off;
 *   "typed"   1 (default) real / imaginary typed records when a matrix has them;
 *   "pdl"     1 (default) programmatic dependent launch of the step kernels.
 *   "narrow"  1 (default) n_b = 2 / 4 / 8 / 12 / 16 whole-row panels of matrices whose every
 *             chunk is one typed record with a staging plan run the narrow
 *             chunk-staged kernel (4 / 4 / 4 / 2 / 2 chunks per stage); 0 = the
 *             register-gather kernel.  (CHEBFD_NARROW)
 *   "npf"    -1 (default) narrow kernel: L2 prefetch of the epilogue rows this many
 *             stages ahead; -1 = 1 for n_b = 12 / 16 except the no-X-update steps, else 0.
 *             (CHEBFD_NPF)
 *   "gpf"     4 (default) register-gather kernel: L2 prefetch distance (blocks) of
 *             generic blocks' U rows (general sparsity); 0 off.
 *   "ko"      0 (default) knock-out bits for bound-finding experiments only
 *             (results are wrong when bits 1-32 are set; bits 64 / 256 / 512 only
 *             reorder work for A/B runs; profiles/producer_ab_r02.md).
 * The same knobs read CHEBFD_STAGED, CHEBFD_NARROW, CHEBFD_X_GROUP, CHEBFD_WPF, CHEBFD_TYPED,
 * CHEBFD_PDL, CHEBFD_GPF from the environment at first use.  Environment only:
 * CHEBFD_FILTER_WIDE=0 (apply_filter keeps n_b != 32 panels as they are instead
 * of filtering them as 32-wide panels), CHEBFD_SOLVE_WIDE=0 (chebfd_solve keeps
 * the caller's n_b for its own block). */
int cf_tuning(const char* key, int value);
/* The calling thread's current CUDA device (cudaGetDevice): the device the
 * C++ drop-in header places matrices and panels on unless chebfilter::set_device
 * selected another one for the thread. */
int cf_current_device(int* device);
int cf_dev_alloc(int device, size_t bytes, void** out);
int cf_dev_free(void* p);
int cf_memcpy(void* dst, const void* src, size_t bytes, int kind);
/* Asynchronous copy on `stream` (cudaMemcpyDefault: host, device or peer memory). */
int cf_memcpy_async(void* dst, const void* src, size_t bytes, void* stream);
int cf_memset_zero(void* p, size_t bytes);
int cf_synchronize(void);

/* ---------------------------------------------------- device kernels ----
 * Raw device pointers to complex128 panels with row stride ld (elements);
 * ncols columns starting at the pointer.  stream: a cudaStream_t (NULL =
 * legacy default stream).  Asynchronous; errors of the launch are returned. */
/* spmmv_shifted (kernels.hpp:82-101): Y = (alpha H + beta) X */
int cf_spmmv_shifted(cf_matrix m, double alpha, double beta, const void* X, void* Y, size_t ld, size_t ncols,
                     void* stream);
/* spmmv_shifted_two_minus (kernels.hpp:104-127): Y = 2(alpha H + beta) X - Z; Z may equal Y */
int cf_spmmv_shifted_two_minus(cf_matrix m, double alpha, double beta, const void* X, void* Y, const void* Z,
                               size_t ld, size_t ncols, void* stream);
/* cheb_init (kernels.hpp:133-152): U = (aH+b)X0; W = 2(aH+b)U - X0; X = g0c0 X0 + g1c1 U + g2c2 W */
int cf_cheb_init(cf_matrix m, double alpha, double beta, void* X, void* U, void* W, size_t ld, size_t ncols,
                 double g0c0, double g1c1, double g2c2, void* stream);
/* Second half of cheb_init as the distributed init runs it after the U halo
 * exchange (dist.hpp:257-262): W = 2(aH+b)U - X; X = g0c0 X + g1c1 U + g2c2 W, fused. */
int cf_cheb_init_tail(cf_matrix m, double alpha, double beta, void* X, const void* U, void* W, size_t ld, size_t ncols,
                      double g0c0, double g1c1, double g2c2, void* stream);
/* chebfd_op (kernels.hpp:160-208): fused W = 2(aH+b)U - W, X += gc W, and
 * eta[j] += <w_new_j, u_j>, mu[j] += <u_j, u_j> into the ncols complex device
 * slots eta, mu (one MomentSeries row at its column offset, :199-202). */
int cf_chebfd_op(cf_matrix m, double alpha, double beta, const void* U, void* W, void* X, size_t ld, size_t ncols,
                 double gc, void* eta, void* mu, void* stream);
/* chebfd_op with the caller's MomentSeries row in HOST memory (the drop-in
 * chebfilter::chebfd_op, kernels.hpp:160-208): the step's moments are reduced
 * into per-matrix device slots (allocated once, zeroed on the stream), read back
 * through a per-matrix pinned buffer and added to eta[j], mu[j] on the host
 * (out += partial, :199-202).  No allocation after the first call; one stream
 * synchronisation (the host row must hold the result on return). */
int cf_chebfd_op_host_moments(cf_matrix m, double alpha, double beta, const void* U, void* W, void* X, size_t ld,
                              size_t ncols, double gc, double* eta, double* mu, void* stream);
/* Fused halo exchange ("mirror"): the same kernels, whose output rows
 * [row_begin, row_end) are ALSO stored to dst + (row - row_begin) * ld -- a
 * neighbour shard's halo slots in peer memory (NVLink) -- so halo_exchange
 * (dist.hpp:110-144) of the next degree's U travels with the step's own stores
 * instead of a separate send/recv.  At most 4 runs per launch. */
typedef struct cf_mirror {
    uint64_t row_begin, row_end; /* output rows, [begin, end) */
    void* dst;                   /* element (row_begin, 0) of the destination panel (same ld) */
} cf_mirror;
int cf_spmmv_shifted_mirror(cf_matrix m, double alpha, double beta, const void* X, void* Y, size_t ld, size_t ncols,
                            const cf_mirror* mir, size_t nmir, void* stream);
int cf_cheb_init_tail_mirror(cf_matrix m, double alpha, double beta, void* X, const void* U, void* W, size_t ld,
                             size_t ncols, double g0c0, double g1c1, double g2c2, const cf_mirror* mir, size_t nmir,
                             void* stream);
int cf_chebfd_op_mirror(cf_matrix m, double alpha, double beta, const void* U, void* W, void* X, size_t ld,
                        size_t ncols, double gc, void* eta, void* mu, const cf_mirror* mir, size_t nmir,
                        void* stream);
/* The degree loop of apply_filter as grouped steps (filter.hpp:87-91 with X
 * updated once per three degrees): step i computes degree[i]
 * with kind[i] = 0 plain chebfd_op (x += gc w_new), 1 no X update, 2 x += gu u
 * + gc w_new, 3 x += gw w_old + gu u + gc w_new.  degree == NULL sizes it.
 * cf_chebfd_step_mirror runs one such step (the distributed drivers' loop). */
int cf_degree_schedule(size_t np, const double* c, const double* g, size_t cap, size_t* count, uint64_t* degree,
                       int* kind, double* gw, double* gu, double* gc);
int cf_chebfd_step_mirror(cf_matrix m, int kind, double alpha, double beta, const void* U, void* W, void* X, size_t ld,
                          size_t ncols, double gw, double gu, double gc, void* eta, void* mu, const cf_mirror* mir,
                          size_t nmir, void* stream);
/* cf_chebfd_step_mirror that also raises `value` in each of the nflags 64-bit
 * flags (neighbours' step-flag slots, cf_flag_signal) once this step's boundary
 * rows are stored (mirrored) and its halo rows read.  With a boundary declared
 * (cf_matrix_set_boundary, boundary-first work order) and the chunk-staged kernel
 * (nflags <= 2), the kernel stores the flags itself as soon as its boundary units
 * are done, while the interior still runs (*in_kernel = 1); otherwise a stream
 * write after the step does (*in_kernel = 0). */
int cf_chebfd_step_signal(cf_matrix m, int kind, double alpha, double beta, const void* U, void* W, void* X, size_t ld,
                          size_t ncols, double gw, double gu, double gc, void* eta, void* mu, const cf_mirror* mir,
                          size_t nmir, void* const* flags, size_t nflags, uint64_t value, void* stream,
                          int* in_kernel);
/* Peer memory between processes (one per GPU): 64-byte cudaIpcMemHandle of a
 * device allocation, opened in another process; and direct peer access for
 * shards of one process on several GPUs. */
int cf_ipc_get_handle(void* dev_ptr, void* handle64);
int cf_ipc_open_handle(int device, const void* handle64, void** dev_ptr);
int cf_ipc_close(void* dev_ptr);
int cf_enable_peer_access(int device, int peer);
/* Per-neighbour step flags, the device-side barrier of the fused halo exchange
 * (replaces a global collective per step; dist.hpp:110-144's init/finalize pair
 * collapses to "my step k is done" / "wait for each neighbour's step k").
 * cf_flag_signal: after the stream's earlier work (with a memory barrier, so the
 * step's mirrored peer stores are visible first) write `value` to the 64-bit
 * `flag`, typically a slot in a neighbour's flag array opened with
 * cf_ipc_open_handle.  cf_flag_wait: the stream waits until the local 64-bit
 * `flag` >= value (no SM is held).  Driver stream memory operations. */
int cf_flag_signal(void* flag, uint64_t value, void* stream);
int cf_flag_wait(const void* flag, uint64_t value, void* stream);
/* apply_filter (filter.hpp:76-93) on a device-resident block vector given as
 * npanels panel pointers (each >= n rows x nb, row stride nb); n_s = npanels*nb.
 * eta, mu: device arrays of (np-2)*n_s complex, index (p-3)*n_s + j (zeroed by
 * the callee).  Scratch U, W panels are owned by the matrix handle. */
int cf_apply_filter(cf_matrix m, void* const* panels, size_t npanels, size_t nb, size_t np, const double* c,
                    const double* g, double alpha, double beta, void* eta, void* mu, void* stream);
/* Same with HOST buffers (X in/out n x n_s panel-concatenated; eta, mu out):
 * the end-to-end entry a CPU caller of apply_filter swaps in.  Panels are
 * host-staged: the device holds two panel slots (not X), panel b+1 is copied in
 * and b-1 out on their own streams while b filters, so X may exceed device
 * memory (cfg3, n_s = 128, on one GPU).  Pinned X (cudaHostAlloc /
 * cudaHostRegister) lets the copies overlap; pageable X is correct but the
 * copies serialise.  Blocking: returns when X and the moments are on the host. */
int cf_apply_filter_host(cf_matrix m, double* X, size_t ns, size_t nb, size_t np, const double* c, const double* g,
                         double alpha, double beta, double* eta, double* mu);

/* filter_distributed (dist.hpp:227-359) for the shards of one process: shard w
 * lives on local's device (shards may share a device), its panels hold
 * local_n owned rows + halo_n halo slots (dist.hpp:88-91), and its send / recv
 * plans are cf_shard's (neighbour, count, rows...) records.  mode 0 = vector
 * (Alg. 3, panel by panel), 1 = pipelined (Alg. 4, degree-major).  Halo rows
 * travel with the kernels' stores into the neighbours' slots over peer memory
 * (or a push kernel for plans of more than 4 runs); X is updated in place in
 * the shards' owned rows; eta, mu: HOST arrays of (np-2)*n_s complex, the
 * worker moments summed in the rank-ordered tree of dist.hpp:344-351. */
typedef struct cf_dist_worker {
    cf_matrix local;          /* shard matrix: local_n rows, local_n + halo_n columns */
    size_t local_n, halo_n;
    void* const* X_panels;    /* n_s/n_b device panels of (local_n + halo_n) x n_b */
    const uint64_t* send_flat;
    size_t send_len;
    const uint64_t* recv_flat;
    size_t recv_len;
} cf_dist_worker;
int cf_filter_distributed(const cf_dist_worker* workers, size_t nworkers, size_t ns, size_t nb, size_t np,
                          const double* c, const double* g, double alpha, double beta, int mode, double* eta,
                          double* mu);

/* cf_filter_distributed with the shards' X panels in HOST memory (X_panels:
 * n_s/n_b host panels of (local_n + halo_n) x n_b; only the owned rows are read
 * and written).  The paper's slow-memory scheme per shard:
 * two device panel slots, panel b+1's owned rows copied in and panel b-1's out
 * on their own streams while panel b filters, so a shard's X may exceed device
 * memory (configs[3]: 137 GB of X per GPU at 8 GPUs).  Vector mode (Alg. 3,
 * dist.hpp:268-282) only: mode 1 fails with CF_EINVAL.  Pinned host panels let
 * the copies overlap the filter.  The device budget (two slots + U/W + moments
 * per shard) is checked up front (CF_EINVAL, never an allocator failure). */
int cf_filter_distributed_host(const cf_dist_worker* workers, size_t nworkers, size_t ns, size_t nb, size_t np,
                               const double* c, const double* g, double alpha, double beta, int mode, double* eta,
                               double* mu);

/* cf_filter_distributed (host_panels 0) or cf_filter_distributed_host (1) with the
 * MEASURED timeline of the degree loop (DistributedResult::timelines,
 * dist.hpp:146-162, 216-219, which the reference fills from a cost model): per
 * worker and (panel, degree) step one "comm" row (the stream waiting for the
 * neighbours' previous steps) and one "compute" row (the step's kernels, halo
 * stores included), from CUDA events.  timeline: cap rows of 6 doubles
 * {worker, kind (0 compute, 1 comm), block, degree, start_ms, end_ms}, times
 * relative to the worker's first event; *count = rows produced (may exceed cap). */
int cf_filter_distributed_timeline(const cf_dist_worker* workers, size_t nworkers, size_t ns, size_t nb, size_t np,
                                   const double* c, const double* g, double alpha, double beta, int mode,
                                   int host_panels, double* eta, double* mu, double* timeline, size_t cap,
                                   size_t* count);

/* stream_bench (perf_model.hpp:80-121) on the device: kind 0 copy, 1 scale,
 * 2 add, 3 triad over `elems` doubles per array; best bytes/s of `reps`. */
int cf_stream_bench(int device, size_t elems, int kind, size_t reps, double* bytes_per_s);

/* --------------------------------------------------- eigensolver (ChebFD) ---
 * The restarted filter loop of chebfd_solve (filter.hpp:247-320): device
 * apply_filter, SVQB orthogonalization (filter.hpp:98-150) and Rayleigh-Ritz
 * (filter.hpp:170-211) with tall-skinny Gram / rotation kernels and a host
 * Jacobi eigensolver on the small projected matrices. */
/* jacobi_hermitian_eig (jacobi_eig.hpp:32-98), host: A k x k row-major complex;
 * values: k ascending; vectors (optional): k x k complex, column j for values[j]. */
int cf_jacobi_hermitian_eig(size_t k, const double* A, double tol, size_t max_sweeps, double* values,
                            double* vectors);
/* S = A^H B (ka x kb, row-major complex, written to the DEVICE buffer S) for
 * device block vectors given as panel pointer lists (element (i, j) of A at
 * a_panels[j / a_nb][i * a_nb + j % a_nb]); ka, kb columns over n rows.  The
 * Gram sums (filter.hpp:99-109, 181-187) in a fixed blocked order. */
int cf_gram(size_t n, void* const* a_panels, size_t a_nb, size_t ka, void* const* b_panels, size_t b_nb, size_t kb,
            void* S, void* stream);
/* Y = A T: A (n x k device panels, width a_nb), T host k x m row-major complex,
 * Y (n x m device panels, width y_nb) -- the rotations of SVQB / Rayleigh-Ritz
 * (filter.hpp:126-135, 193-199) over a shard's own rows. */
int cf_rotate(size_t n, void* const* a_panels, size_t a_nb, size_t k, const double* T, size_t m, void* const* y_panels,
              size_t y_nb, void* stream);
/* Per column r < k: num_den[2r] = sum |HY(i,r) - theta_r Y(i,r)|^2, num_den[2r+1] = sum |Y(i,r)|^2
 * over n rows (filter.hpp:203-209 partial sums; a distributed solve adds them over ranks). */
int cf_residual_sums(size_t n, void* const* y_panels, size_t y_nb, void* const* hy_panels, size_t hy_nb, size_t k,
                     const double* theta, double* num_den, void* stream);
/* orthogonalize_svqb (filter.hpp:139-150): X (n x n_s device panels) ->
 * Q written to the device buffer Q as one n x rank panel (row stride rank;
 * Q must hold n * n_s complex).  drop_tol as the reference (default 1e-12). */
int cf_orthogonalize_svqb(size_t n, void* const* panels, size_t npanels, size_t nb, double drop_tol, void* Q,
                          size_t* rank, void* stream);
/* rayleigh_ritz (filter.hpp:170-211): Q one n x k device panel (row stride k,
 * orthonormal to 1e-8 or CF_EINVAL); theta, residuals: k host doubles
 * (ascending theta); basis: device n x k panel, Y = Q V. */
int cf_rayleigh_ritz(cf_matrix m, const void* Q, size_t k, double* theta, void* basis, double* residuals,
                     void* stream);

/* SolveOptions (filter.hpp:230-241); damping 0 = jackson, 1 = none. */
typedef struct cf_solve_options {
    size_t n_s, n_b, n_p, max_restarts;
    double res_tol, margin;
    uint64_t seed;
    int damping;
    int has_bounds; /* 1: use bound_lo/hi (spectral_bounds), 0: Gershgorin of the matrix */
    double bound_lo, bound_hi;
    double drop_tol;
} cf_solve_options;

/* SolveResult (filter.hpp:220-228).  Caller-owned buffers, each sized n_s
 * unless noted; NULL skips an optional output. */
typedef struct cf_solve_result {
    size_t n_eig;           /* converged in-window pairs */
    size_t n_pairs;         /* pairs of the last Rayleigh-Ritz extraction */
    size_t iterations;      /* restarts run */
    int converged;
    double* eigenvalues;    /* n_eig, ascending */
    double* residuals;      /* n_eig */
    double* pair_values;    /* n_pairs (all_pairs) */
    double* pair_residuals; /* n_pairs */
    int* pair_flags;        /* n_pairs: bit 0 inside_window, bit 1 converged */
    void* eigenvectors;     /* optional DEVICE buffer, n x n_s complex: n x n_eig panel (row stride n_eig) */
    double* eta;            /* optional HOST buffer, max_restarts * (n_p-2) * n_s complex (moments per restart) */
    double* mu;             /* optional HOST buffer, same shape */
    double* phase_ms;       /* optional HOST buffer, max_restarts x 3: per restart the wall time
                               (ms, each phase ends in a stream sync) of the filter, SVQB and
                               Rayleigh-Ritz phases */
} cf_solve_result;

/* chebfd_solve (filter.hpp:247-320) on a device matrix (built from the whole
 * CRS; shard-local matrices are rejected).  Throws CF_EINVAL for a window
 * outside the spectral bounds; non-convergence is reported in res->converged. */
int cf_chebfd_solve(cf_matrix m, double window_lo, double window_hi, const cf_solve_options* opt,
                    cf_solve_result* res, void* stream);

#ifdef __cplusplus
}
#endif
#endif
