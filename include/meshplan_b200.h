/*
 * meshplan_b200.h -- C ABI of the B200-native indirect-increment engine.
 *
 * Plain C: pointers, sizes and PODs only; no torch or C++ types.  Device
 * pointers are CUDA global-memory addresses owned by the caller; `stream`
 * is a cudaStream_t passed as void*.  Every entry point returns an mp_status
 * (0 = ok); the message of the last failure on the calling thread is
 * available from mp_last_error().  The status values follow the reference
 * CLI exit codes (pkg/src/meshplan/cli.py:368-377, errors.py:8-29).
 *
 * Which reference interface each entry point replaces is noted beside it.
 * The reference is pure Python (pkg/src/meshplan); its seams are
 *   Seam A  meshplan._accel  (pkg/src/meshplan/_accel/__init__.py:43-50)
 *   Seam B  the loop/plan API (plan.py:408, plan.py:467, simulator.py:215/355/525)
 * INTEGRATION.md shows the ctypes binding a maintainer would add.
 */
#ifndef MESHPLAN_B200_H
#define MESHPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t mp_status;
enum {
  MP_OK = 0,
  MP_ERR_CUDA = 1,       /* CUDA runtime failure                          */
  MP_ERR_KERNEL = 2,     /* KernelSpecError   (exit code 2)               */
  MP_ERR_RACE = 3,       /* RaceError         (exit code 3)               */
  MP_ERR_CAPACITY = 4,   /* CapacityError     (exit code 4)               */
  MP_ERR_FORMAT = 5,     /* FileFormatError   (exit code 5)               */
  MP_ERR_VALIDATION = 6  /* MeshValidationError (exit code 2)             */
};

enum { MP_F64 = 0, MP_F32 = 1, MP_I64 = 2, MP_I32 = 3 };          /* element types  */
enum { MP_AOS = 0, MP_SOA = 1 };                                   /* array layouts  */
enum {                                                             /* device element ops */
  MP_OP_FLUX = 0,            /* bench_kernels.py:154-189                   */
  MP_OP_FLUX_NOREAD = 1,     /* bench_kernels.py:174-176                   */
  MP_OP_SCATTER8 = 2,        /* bench_kernels.py:192-207                   */
  MP_OP_FACE_FLUX = 3,       /* bench_kernels.py:210-246                   */
  MP_OP_FACE_FLUX_HEAVY = 4  /* bench_kernels.py:234-237                   */
};
enum { MP_SCHED_COLOUR = 0, MP_SCHED_DATAFLOW = 1,                /* hierarchical schedules */
       MP_SCHED_PULL = 4 };  /* | flag, pipelined executor: pull-list form of the colour loop */

/* One indirect loop bound to device arrays (plan numbering).
 * Indirect arrays (ind_read, inc) use ind_layout; direct arrays are SoA
 * (plan.py:381-398).  Element e's slot s point is map[e*arity+s] (AoS) or
 * map[s*n_elems+e] (SoA). */
typedef struct mp_loop {
  int32_t op;            /* MP_OP_*                                        */
  int32_t unit;          /* 1: unit-increment variant (incidence counting)  */
  int32_t dtype;         /* MP_F64 ... shared by every array of the loop   */
  int32_t ind_layout;    /* MP_AOS / MP_SOA                                */
  int64_t n_elems;       /* iteration-set size                             */
  int64_t n_points;      /* to-set size                                    */
  int32_t arity;
  int32_t map_layout;    /* MP_AOS / MP_SOA                                */
  const int32_t* map;
  const void* ind_read;  /* q / state, or NULL                             */
  int32_t ind_read_comps;
  int32_t dir_comps;
  const void* dir_read;  /* w / stress / facew (SoA)                       */
  void* inc;             /* res / force / flux, incremented in place        */
  int32_t inc_comps;
  int32_t pad_;
} mp_loop;

/* Device-resident hierarchical plan (HierarchicalPlan, plan.py:132-185).
 * Blocks are contiguous element ranges; a point's shared slot is its
 * position in the block's ascending staged list (plan.py:168-182),
 * materialised here as local_slots (per element and slot) and
 * written_slots (per written entry). */
typedef struct mp_hier_plan {
  int32_t num_blocks;
  int32_t block_size;           /* widest block (CTA width)                 */
  int32_t stage_reads;          /* 1: all-indirect staging, 0: increment-only */
  int32_t max_staged;           /* widest staged list (shared sizing)        */
  int32_t slot_bytes;           /* 1 (max_staged <= 256) or 2: local_slots width */
  int32_t written_is_staged;    /* 1: every block's written list == staged list */
  const int32_t* meta;            /* [nb][4] {first element, elements,
                                     staged offset, staged count}            */
  const int32_t* staged_ids;      /* ascending per block                     */
  const int32_t* written_offsets; /* [nb+1] (written_is_staged == 0 only)    */
  const int32_t* written_ids;     /* ascending per block                     */
  const uint16_t* written_slots;  /* staged slot of each written entry       */
  const void* local_slots;        /* [n_elems*arity] staged slot per map entry */
  const uint8_t* thread_colours;  /* [n_elems] sorted within each block      */
  const int32_t* colour_counts;   /* [nb] thread colours per block           */
  /* MP_SCHED_COLOUR: one launch per block colour */
  int32_t num_block_colours;
  int32_t pad_;
  const int32_t* colour_block_offsets_host; /* host [ncol+1]                  */
  const int32_t* blocks_by_colour;          /* device [nb], (colour, id) order */
  /* MP_SCHED_DATAFLOW: one launch, blocks in a topological order of the
   * lower-colour conflict DAG; each block waits for its predecessors. */
  const int32_t* order;           /* [nb]                                    */
  const int32_t* pred_offsets;    /* [nb+1]                                  */
  const int32_t* preds;           /* conflicting blocks of lower colour      */
  uint32_t* flags;                /* [nb] epoch stamps, zero-initialised     */
  uint32_t* tickets;              /* [2] next-block ticket, finished blocks;
                                     zero-initialised, re-armed by the kernel */
  /* Pull lists (optional, pipelined executor): for block b and staged row j,
   * the (element*arity + slot) refs writing row j in thread-colour order are
   * pull_ref[e0*arity + pull_off[s0 + b + j] .. pull_off[s0 + b + j + 1]). */
  const uint16_t* pull_off;       /* [staged total + nb] (or NULL)           */
  const uint16_t* pull_ref;       /* [n_elems*arity]                         */
  /* Streamed executor (mp_exec_hier_stream): per-ticket block descriptors
   * {first element, elements | thread colours << 16, staged offset, staged
   * count} in blocks_by_colour order and in dataflow order, and one packed
   * record per element: arity local slots (slot_bytes each), the element's
   * thread colour (1 byte), a mask of the slots through which the element is
   * the first writer of its staged row within the block (1 byte, arity <= 8),
   * zero padding to elem_meta_bytes (multiple of 4). */
  const int32_t* tdesc_colour;    /* [nb][4]                                 */
  const int32_t* tdesc_order;     /* [nb][4]                                 */
  const uint8_t* elem_meta;       /* [n_elems*elem_meta_bytes]               */
  int32_t elem_meta_bytes;
  int32_t pad2_;
  /* predecessor lists re-indexed by dataflow ticket: the preds (block ids)
   * of block order[t] are tpreds[tpred_offsets[t] .. tpred_offsets[t+1]) */
  const int32_t* tpred_offsets;   /* [nb+1]                                  */
  const int32_t* tpreds;
  /* the same lists padded to 8 per ticket: -1 = no predecessor, -2 in slot 7 =
   * the list continues in tpreds (from its 8th entry) */
  const int32_t* tpred_pad;       /* [nb][8]                                 */
  const int32_t* tblock_colour;   /* [nb] block id of each tdesc_colour entry */
} mp_hier_plan;

/* ---- library ------------------------------------------------------------ */
const char* mp_last_error(void);
const char* mp_version(void);
int32_t mp_device_sm_count(int32_t device);

/* ---- executors (Seam B) --------------------------------------------------- */
/* execute_global (simulator.py:355-439): one launch per colour range
 * [colour_offsets[c], colour_offsets[c+1]) (host array), direct non-atomic
 * read-modify-write of inc; bit-exact with the reference colour order. */
mp_status mp_exec_global(const mp_loop* loop, const int64_t* colour_offsets, int32_t num_colours,
                         int32_t block_size, void* stream);

/* execute_hierarchical (simulator.py:525-656): stage, compute, apply
 * increments in shared memory one thread colour at a time, scatter the
 * written list once per block.  `epoch` must increase by one per call on a
 * plan when schedule == MP_SCHED_DATAFLOW (flags are epoch stamps). */
mp_status mp_exec_hier(const mp_loop* loop, const mp_hier_plan* plan, int32_t schedule, uint32_t epoch,
                       void* stream);

/* Same semantics and results as mp_exec_hier, as a persistent
 * warp-specialised kernel: one producer warp per CTA fills a 3-stage
 * mbarrier ring with cp.async gathers (staged ids and rows, increment rows,
 * slots, direct operands, colours) ahead of the consumer warps.  Needs
 * written_is_staged and block_size <= 992.  MP_SCHED_DATAFLOW: the producer
 * acquires the predecessors' flags before gathering increment rows. */
mp_status mp_exec_hier_pipelined(const mp_loop* loop, const mp_hier_plan* plan, int32_t schedule, uint32_t epoch,
                                 void* stream);

/* Same semantics and results as mp_exec_hier, as a lean persistent kernel:
 * every thread both gathers and computes; a D-deep cp.async ring (one commit
 * group per block) keeps D blocks in flight; descriptor -> staged-id -> row
 * loads are software-pipelined in registers; shared rows use a
 * bank-conflict-free odd-granule pitch.  MP_SCHED_DATAFLOW adds a sync warp
 * per CTA that checks predecessors ahead of use and releases finished blocks
 * in batches.  Needs written_is_staged, tdesc_* and elem_meta. */
mp_status mp_exec_hier_stream(const mp_loop* loop, const mp_hier_plan* plan, int32_t schedule, uint32_t epoch,
                              void* stream);

/* Atomics baseline (reference cost model only,
 * simulator.py:331-341): one thread per element in the loop's element order,
 * increments applied with hardware atomics.  Results equal the reference up
 * to floating-point reassociation.  A comparison baseline, not the product. */
mp_status mp_exec_atomic(const mp_loop* loop, void* stream);

/* execute_serial (simulator.py:215-230) on the device: per-element
 * increments to a temp array, then per point an ordered sum over its
 * (element, slot) references (inverse CSR, mesh.py:251-267), i.e. exactly the
 * np.add.at order.  temp must hold n_elems*arity*inc_comps elements. */
mp_status mp_exec_serial(const mp_loop* loop, const int32_t* inv_offsets, const int32_t* inv_refs, void* temp,
                         void* stream);

/* mp_exec_hier_stream (colour schedules) with the multi-GPU halo export
 * fused into the write-back.  export_desc: device memory holding
 *   { const int32_t* dest;            per staged entry: (peer << 24 | row) for
 *                                     the halo rows whose block is their last
 *                                     writer, -1 elsewhere
 *     uint64_t base[8];               per peer: the owner's export mailbox slot
 *                                     for this rank (parity 0), IPC-mapped
 *     int64_t stride[8];              bytes between its two parity slots
 *     const uint32_t* epoch; }        the device step epoch (parity = epoch & 1)
 * (mp_export_desc_bytes() = its size).  The last writer of a halo row also
 * stores the row's final value into row `row` of base[peer] + parity *
 * stride[peer] (P2P stores over NVLink). */
mp_status mp_export_desc_bytes(void);
mp_status mp_exec_hier_stream_export(const mp_loop* loop, const mp_hier_plan* plan, int32_t schedule,
                                     const void* export_desc, void* stream);

/* Hierarchical executor, gather form (colour schedule, one launch per block
 * colour): lanes own (element, slot) refs instead of elements; each row's
 * refs are summed in thread-colour order by a shuffle chain and written back
 * once -- bit-identical to mp_exec_hier_stream and execute_hierarchical
 * (simulator.py:525-656) on the same plan, without the thread-colour loop.
 * ref_offsets / refs from mp_plan_gather_refs; max_refs = the widest block's
 * position count.  AoS indirect arrays, staged reads. */
mp_status mp_exec_hier_gather(const mp_loop* loop, const mp_hier_plan* plan, const int32_t* ref_offsets,
                              const uint32_t* refs, int32_t max_refs, void* stream);

/* ---- multi-GPU halo (owner compute; no reference counterpart) ----- */
/* dst[r*comps + c] = src[rows[r]*comps + c]  (pack rows a peer imports)      */
mp_status mp_halo_pack(int32_t dtype, const void* src, const int32_t* rows, int64_t nrows, int32_t comps, void* dst,
                       void* stream);
/* dst[rows[r]*comps + c] = src[r*comps + c] (mode 0), += (mode 1, fold a peer's
 * increments), = 0 (mode 2, re-zero halo increments); rows distinct */
mp_status mp_halo_unpack(int32_t dtype, void* dst, const int32_t* rows, int64_t nrows, int32_t comps,
                         const void* src, int32_t mode, void* stream);

/* Peer-memory halo exchange (graph-capturable, no NCCL on the data path).
 * put: rows of src -> the receiver's mailbox slot (remote: an IPC-mapped or
 * same-device pointer; slot = epoch parity, slot_elems apart), then
 * *remote_flag = epoch once all stores are visible system-wide (done_counter:
 * a zeroed device word private to this put).  get: wait until *flag reaches
 * the epoch, then dst rows = (mode 0) / += (mode 1) the mailbox slot.  The
 * epoch is read from device memory at kernel start; mp_epoch_bump adds 1. */
mp_status mp_halo_put(int32_t dtype, const void* src, const int32_t* rows, int64_t nrows, int32_t comps, void* remote,
                      int64_t slot_elems, uint32_t* remote_flag, const uint32_t* epoch, uint32_t* done_counter,
                      void* stream);
mp_status mp_halo_get(int32_t dtype, void* dst, const int32_t* rows, int64_t nrows, int32_t comps, const void* mailbox,
                      int64_t slot_elems, const uint32_t* flag, const uint32_t* epoch, int32_t mode, void* stream);
mp_status mp_epoch_bump(uint32_t* epoch, void* stream);
/* Release the step epoch into a peer's flag after this stream's earlier work
 * (the fused export's P2P row stores) -- the put without the copy. */
mp_status mp_halo_signal(uint32_t* remote_flag, const uint32_t* epoch, void* stream);
/* Zeroed device allocation (cudaMalloc: IPC-exportable; free with mp_free),
 * its 64-byte IPC handle, and a peer process's mapping of one (closed with
 * mp_ipc_close). */
mp_status mp_mailbox_alloc(int64_t bytes, void** ptr);
mp_status mp_ipc_handle(void* ptr, unsigned char* handle);
mp_status mp_ipc_open(const unsigned char* handle, void** ptr);
mp_status mp_ipc_close(void* ptr);

/* ---- race checks (simulator.py:245-261, 446-469) ---------------------------- */
/* Keys (group*key_span + point) over every (element, written point) ref;
 * returns in first_pair[0..1] the first pair of distinct elements sharing a
 * key in (key, element) order, or -1/-1.  refs are per-element CSR. */
mp_status mp_race_check(int64_t n_items, const int64_t* ref_offsets, const int32_t* refs, const int64_t* groups,
                        int64_t key_span, int64_t* first_pair, void* stream);

/* ---- planner kernels ------------------------------------------------------ */
/* Per block: ascending unique points referenced through the slots in
 * slot_mask.  Pass 1 (ids == NULL): counts[b].  Pass 2: fill ids at
 * offsets[b].  (plan.py:582-603) */
mp_status mp_plan_block_points(int32_t nb, const int32_t* block_offsets, const int32_t* map, int64_t n_elems,
                               int32_t arity, int32_t map_layout, uint32_t slot_mask, int32_t max_block,
                               int32_t* counts, const int32_t* offsets, int32_t* ids, void* stream);

/* local_slots[e*arity+s] = position of map(e,s) in block's ids list (binary
 * search); written_slots likewise for a second list.  Returns
 * MP_ERR_CAPACITY when a point is missing (plan.py:168-182). */
mp_status mp_plan_local_slots(int32_t nb, const int32_t* block_offsets, const int32_t* map, int64_t n_elems,
                              int32_t arity, int32_t map_layout, uint32_t slot_mask, const int32_t* staged_offsets,
                              const int32_t* staged_ids, uint16_t* local_slots, const int32_t* written_offsets,
                              const int32_t* written_ids, uint16_t* written_slots, void* stream);

/* Per-block thread colouring (plan.py:260-284): conflict graph of elements
 * sharing a written point, smallest-last order (numpy_impl.py:95-111,
 * key deg*(k+1)+u), first-fit greedy (numpy_impl.py:62-92).  Outputs the
 * unsorted colour of each element, the colour count per block, and the
 * stable colour sort as local order (plan.py:508-517). */
mp_status mp_plan_thread_colours(int32_t nb, const int32_t* block_offsets, const int32_t* map, int64_t n_elems,
                                 int32_t arity, int32_t map_layout, uint32_t written_mask, int32_t max_block,
                                 int32_t* colours, int32_t* counts, int32_t* sorted_order, void* stream);

/* Gather-form ref records (see mp_exec_hier_gather): pass 1 (refs == NULL)
 * writes per-block position counts; the caller scans them into ref_offsets
 * [nb+1], fills refs with 0xFF bytes and calls again.  Built from the plan's
 * pull lists (mp_hier_plan.pull_off / pull_ref). */
mp_status mp_plan_gather_refs(int32_t nb, const int32_t* block_offsets, const int32_t* staged_offsets,
                              const uint16_t* pull_off, const uint16_t* pull_ref, int32_t arity,
                              const int32_t* ref_offsets, int32_t* counts, uint32_t* refs, void* stream);

/* Executor layout of each block's staged rows (not part of the plan):
 * perm[staged_offsets[b] + position] = staged index placed at that shared
 * row, chosen so that each quarter-warp access group (colour-loop
 * read-modify-writes, element reads; thread_colours colour-sorted per block)
 * touches rows in distinct classes mod 8, i.e. distinct 16-byte bank groups.
 * local_slots: per (element, slot) staged index, 0xFFFF when not staged. */
mp_status mp_plan_row_placement(int32_t nb, const int32_t* block_offsets, const int32_t* staged_offsets,
                                const uint16_t* local_slots, int32_t arity, const uint8_t* thread_colours,
                                int32_t* perm, void* stream);

/* Greedy colouring of the plan blocks over their written points, on the
 * device (replaces _accel.greedy_colour_csr at plan.py:254 in
 * _colour_blocks_ns, plan.py:241-257): bit-identical to greedy_colour_csr
 * (numpy_impl.py:12-60) with blocks as items, least-loaded or first-fit,
 * before the relabel by load.  written_offsets/ids: per-block ascending
 * unique written points (device int32 CSR, mp_plan_block_points); colours:
 * device int32[nb]; *num_colours (host) receives the colour count.  Lower-id
 * conflict lists are built by sorts; one warp then walks the blocks in order.
 * MP_ERR_CAPACITY beyond 1024 colours. */
mp_status mp_plan_block_colours(int32_t nb, const int32_t* written_offsets, const int32_t* written_ids,
                                int32_t least_loaded, int32_t* colours, int32_t* num_colours, void* stream);

/* Sequential greedy colouring of items over shared points, host C++,
 * bit-identical to greedy_colour_csr (numpy_impl.py:12-60). */
mp_status mp_greedy_colour_csr(int64_t n_items, const int64_t* indptr, const int64_t* indices, int64_t n_points,
                               int32_t least_loaded, int64_t* colours);

/* First-fit / least-loaded greedy over an adjacency CSR in a given order
 * (numpy_impl.py:62-92), host C++. */
mp_status mp_greedy_colour_adj(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* order,
                               int32_t least_loaded, int64_t* colours);

/* Smallest-last elimination order (numpy_impl.py:95-111), host C++. */
mp_status mp_smallest_last_order(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t* order);

/* Multilevel k-way partitioner pieces (partition.py:173-350), host C++,
 * bit-identical to the reference's sequential sweeps.  CSR graphs are int64
 * host arrays; `assignment` / `block_w` are updated in place. */
mp_status mp_heavy_edge_matching(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* weights,
                                 const int64_t* node_w, const int64_t* visit, int64_t max_cluster, int64_t* match);
mp_status mp_cut_weight(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* weights,
                        const int64_t* assignment, int32_t use_w, int64_t* cut);
mp_status mp_refine_boundary_pass(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* weights,
                                  int64_t* assignment, int64_t* block_w, int64_t num_blocks, const int64_t* node_w,
                                  int64_t cap, int32_t use_w, int64_t* moves);
/* Up to `max_passes` of those sweeps, stopping after one with no move
 * (partition.py:326-337); later sweeps visit only the nodes whose decision can
 * change.  `moves` receives the total over all sweeps. */
mp_status mp_refine_boundary(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* weights,
                             int64_t* assignment, int64_t* block_w, int64_t num_blocks, const int64_t* node_w,
                             int64_t cap, int32_t use_w, int32_t max_passes, int64_t* moves);
mp_status mp_rebalance(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* weights,
                       int64_t* assignment, int64_t* block_w, int64_t num_blocks, const int64_t* node_w, int64_t cap,
                       int32_t use_w);
mp_status mp_initial_partition(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* node_w,
                               int64_t num_blocks, int64_t cap, int64_t* assignment);

/* mp_heavy_edge_matching on device arrays (numpy_impl.py:134-157; replaces
 * _accel.heavy_edge_matching at partition.py:317): the same matching as the
 * sequential visit-order greedy, computed in dependency rounds (a node acts
 * once every earlier-visited node within two hops is matched).  `rounds`
 * receives the number of rounds; after 4096 rounds (MESHPLAN_MATCH_ROUNDS)
 * the remaining turns finish on the host, still exact, and `rounds` is
 * negated. */
mp_status mp_heavy_edge_matching_device(int32_t n, const int64_t* indptr, const int64_t* indices,
                                        const int64_t* weights, const int64_t* node_w, const int64_t* visit,
                                        int64_t max_cluster, int64_t* match, int32_t* rounds, void* stream);

/* Level-synchronous BFS on a device CSR graph (numpy_impl.py:114-131):
 * levels[v] (-1 unreached); returns the eccentricity and visited count.
 * Levels are independent of visit order, so equal to the reference. */
mp_status mp_bfs_levels(int32_t n, const int64_t* indptr, const int32_t* indices, int32_t start, int32_t* levels,
                        int32_t* ecc, int32_t* visited, void* stream);

/* Host BFS with the reference's outputs (numpy_impl.py:114-131; replaces
 * _accel.bfs_levels, reorder.py:101/106/127/131): levels[n] (-1 unreached),
 * the FIFO visit queue[n] (first *tail entries valid) and *tail. */
mp_status mp_bfs_levels_host(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t start,
                             int64_t* levels, int64_t* queue, int64_t* tail);

/* All unordered pairs within each CSR segment, as (min, max)
 * (numpy_impl.py:231-259; replaces _accel.pairs_from_segments,
 * reorder.py:78, colouring.py:138, partition.py:82).  Pair order is
 * unspecified in the reference; here segment by segment, (i, j) position
 * order.  us == NULL: only *num_pairs (the size) is written. */
mp_status mp_pairs_from_segments(int64_t num_segments, const int64_t* seg_indptr, const int64_t* seg_values,
                                 int64_t* us, int64_t* vs, int64_t* num_pairs);

/* Block conflict DAG for the dataflow schedule: for every pair of blocks
 * writing a common point, an edge from the lower to the higher
 * (colour, id); order = blocks sorted by (key, id) where
 * key(b) = max(b, max_pred key+1), a topological order close to id order. */
mp_status mp_plan_block_dag(int32_t nb, const int32_t* written_offsets, const int32_t* written_ids,
                            int64_t n_points, const int32_t* block_colours, int32_t num_colours, int32_t lag,
                            int32_t* pred_offsets /* [nb+1] */, int32_t* preds, int64_t preds_capacity,
                            int64_t* num_preds, int32_t* order, void* stream);
/* (when *num_preds > preds_capacity nothing but *num_preds is written:
 *  grow the buffer and call again) */
void mp_free(void* device_ptr);

#ifdef __cplusplus
}
#endif
#endif /* MESHPLAN_B200_H */
