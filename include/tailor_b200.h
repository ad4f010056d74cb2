/*
 * tailor_b200.h — C ABI of the B200-native checkpoint-tailoring hot path.
 *
 * The reference (LLMTailor C++ library, /root/reference/proj) exposes this
 * path only as C++ (R/include/tailor/merge.hpp, R/include/tailor/recipe.hpp)
 * and as the `tailor merge` / `tailor plan` CLI; it has no FFI. These entry
 * points are what a binding of that path (ctypes, cgo, JNI) needs: plain
 * pointers, sizes and int codes; no C++ or torch types, no exceptions.
 * Each function cites the reference interface it replaces.
 *
 * Errors: every int-returning function returns TG_OK (0) or the reference's
 * ErrorKind code below; tg_last_error() holds the message (thread-local).
 * User errors (codes 1..9) are the reference's exit-code-1 class; 10, 11, 12
 * and 100 are internal (exit 2), as R/include/tailor/errors.hpp:51-54.
 * A null handle passed to an int-returning function is TG_E_GEOMETRY ("<fn>: null
 * handle"); size/count getters return 0 for a null handle.
 *
 * Device pointers are CUDA global-memory addresses on the current device;
 * `stream` is a cudaStream_t (NULL = legacy default stream). Launches are
 * asynchronous on that stream; the caller synchronizes.
 */
#ifndef TAILOR_B200_H
#define TAILOR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    TG_OK = 0,
    TG_E_INVALID_MODULE = 1,
    TG_E_GEOMETRY = 2,
    TG_E_NON_FINITE = 3,
    TG_E_RECIPE = 4,
    TG_E_SOURCE_LACKS_MODULE = 5,
    TG_E_MISSING_ARTIFACT = 6,
    TG_E_CORRUPT_CONTAINER = 7,
    TG_E_UNRECOVERABLE_MODULE = 8,
    TG_E_MISSING_MODULES = 9,
    TG_E_CONSISTENCY = 10,
    TG_E_STORAGE = 11,
    TG_E_DEVICE = 12,
    TG_E_INTERNAL = 100
};

/* ModelSpec (R/include/tailor/model.hpp:14-30). */
typedef struct tg_model_spec {
    int32_t num_layers;
    int32_t hidden_dim;
    int32_t ffn_dim;
    int32_t vocab_size;
    int32_t weight_tied;
    int32_t reserved;
    uint64_t seed;
} tg_model_spec;

/* MergeOptions / MergeStats (R/include/tailor/merge.hpp:46-55), extended with
 * device timing, the composite byte count, the devices the output lanes run on and
 * the file I/O mode. A zero-initialised struct means: workers = default, cached,
 * device 0, re-verify on (the reference always re-verifies, R/src/merge.cpp:353),
 * io_mode auto. */
enum {
    TG_IO_AUTO = 0,        /* O_DIRECT reads of source files mostly absent from the page cache */
    TG_IO_BUFFERED = 1,    /* everything through the page cache (the reference's behaviour) */
    TG_IO_DIRECT = 2,      /* O_DIRECT reads of every source file */
    TG_IO_DIRECT_RW = 3    /* + O_DIRECT writes of the output files */
};
typedef struct tg_merge_options {
    int32_t workers;        /* output/IO lanes; 0 = max(num_ranks, host threads) */
    int32_t uncached;       /* reload source shard per group copy (benchmark mode) */
    int32_t device;         /* the device of every lane when num_devices == 0 */
    int32_t skip_verify;    /* 1 = skip the device re-verify of the written composite */
    const int32_t* devices; /* num_devices > 0: lanes spread round-robin over devices[0..num_devices);
                               output bytes do not depend on the devices (R/tests/acceptance.cpp:442-458) */
    int32_t num_devices;
    int32_t io_mode;        /* TG_IO_*; the TAILOR_IO environment variable overrides it */
} tg_merge_options;

typedef struct tg_merge_stats {
    int64_t shard_files_read;
    int64_t weight_files_read;
    double wall_ms;
    double device_ms;
    uint64_t bytes_moved;
    uint64_t direct_read_bytes;  /* source bytes read with O_DIRECT */
    uint64_t direct_write_bytes; /* output bytes written with O_DIRECT (whole 4 KB blocks) */
    uint64_t resident_bytes;     /* source bytes gathered from device copies instead of read (tg_select_merge) */
} tg_merge_stats;

/* K2 segment: dst[dst_off, dst_off+bytes) <- src[0, bytes). */
typedef struct tg_gather_seg {
    const uint8_t* src;
    uint64_t dst_off;
    uint64_t bytes;
} tg_gather_seg;

/* K3 tile over `count` master elements of field `field` of module `module`. */
typedef struct tg_score_tile {
    uint32_t module;
    uint32_t field;
    uint32_t count;
    uint32_t pad;
    uint64_t elem_start;
} tg_score_tile;

typedef struct tg_layout tg_layout;
typedef struct tg_family tg_family;
typedef struct tg_scorer tg_scorer;
typedef struct tg_mplan tg_mplan;

/* ---- errors / info ---------------------------------------------------------- */
const char* tg_last_error(void);
int tg_last_error_kind(void);
const char* tg_version(void);
int tg_device_count(void);

/* ---- L5 drop-ins on checkpoint directories ------------------------------------
 * Text outputs (JSON / YAML) use the (buf, cap, needed) convention: `needed`
 * receives strlen+1; the call fails with TG_E_GEOMETRY if cap is too small. */

/* parse_recipe (R/src/recipe.cpp:67-132) -> recipe as JSON. */
int tg_parse_recipe(const char* yaml, char* json_out, size_t cap, size_t* needed);
/* recipe_to_yaml (R/src/recipe.cpp:139-169) of a JSON recipe. */
int tg_recipe_to_yaml(const char* recipe_json, char* yaml_out, size_t cap, size_t* needed);
/* resolve_plan (R/src/merge.cpp:39-152) -> MergePlan as JSON. */
int tg_resolve_plan(const char* recipe_yaml, char* plan_json, size_t cap, size_t* needed);
/* cmd_merge -> execute_merge (R/tools/tailor_main.cpp:75-103, R/src/merge.cpp:226-357). */
int tg_execute_merge(const char* recipe_yaml, const char* out_dir, const tg_merge_options* options,
                     tg_merge_stats* stats);
/* recipe_from_manifests (R/src/merge.cpp:359-418) -> recipe YAML. */
int tg_recipe_from_manifests(const char* run_dir, int64_t failure_step, char* yaml_out, size_t cap, size_t* needed);
/* coarse_to_fine / fine_to_coarse of a complete checkpoint directory (R/src/groups.cpp:152-220
 * between read_checkpoint and write_checkpoint), as a device gather: to_fine=1 -> 2L+3 groups. */
int tg_regroup(const char* src_dir, const char* out_dir, int32_t to_fine, const tg_merge_options* options,
               tg_merge_stats* stats);
/* Device-resident trainer: train() (R/src/trainer.cpp:109-123) with the
 * optimizer state in HBM and bit-exact AdamW (R/src/adamw.cpp:10-66); strategy 0 full,
 * 1 parity, 2 filter (R/src/strategy.cpp:48-91), 3 magnitude (in-situ update-magnitude
 * selection, rho = fraction of modules saved per checkpoint after the first). */
typedef struct tg_train_config {
    int32_t total_steps;
    int32_t num_ranks;
    int32_t interval;
    int32_t strategy;
    int32_t head_count;
    int32_t tail_count;
    int32_t sparse_multiple;
    int32_t device;
    double lr;
    double weight_decay;
    double rho;
} tg_train_config;
int tg_train(const tg_model_spec* spec, const tg_train_config* config, const char* out_dir,
             int32_t* checkpoints_written);
/* resume (R/src/trainer.cpp:125-152) on the device: verify a complete fine checkpoint,
 * continue `additional_steps` steps with its strategy, rank count and per-group
 * hyperparameters, writing checkpoints + log.jsonl into a fresh out_dir. */
int tg_resume(const char* checkpoint_dir, int64_t additional_steps, const char* out_dir, int32_t device,
              int32_t* checkpoints_written);
/* A resident trainer over rank partitions [rank_begin, rank_end) of a num_ranks layout
 * (one per GPU in a ZeRO job): train_step (R/src/trainer.cpp:26-35) on the device. */
typedef struct tg_trainer tg_trainer;
tg_trainer* tg_trainer_create(const tg_model_spec* spec, int32_t num_ranks, int32_t rank_begin, int32_t rank_end, double lr,
                              double weight_decay, int32_t device);
void tg_trainer_destroy(tg_trainer* t);
uint64_t tg_trainer_elements(const tg_trainer* t);
int tg_trainer_step(tg_trainer* t, int64_t step, double* grad_norm, double* update_norm);
/* Device pointer and byte size of rank partition `rank` (optim/rank_<rank>.shard payload
 * layout); valid until the trainer is destroyed. */
int tg_trainer_partition(tg_trainer* t, int32_t rank, void** d_ptr, uint64_t* bytes);
/* read_checkpoint's invariants (R/src/checkpoint.cpp:485-575), checked on the device. */
int tg_verify_checkpoint(const char* dir, int32_t device);
/* Update-magnitude scores of consecutive snapshot directories on the device
 * (SURVEY §8 a13): sums[(p*M + m)*2 + {0,1}] = (sum delta^2, sum ref^2) of
 * pair p = (dirs[p], dirs[p+1]); scores[p*M + m]. Capacity: (n-1)*M. Any n >= 2.
 * Rank partitions are scored by lanes spread over devices[0..num_devices)
 * (NULL / 0 = device 0) and combined in rank order: results do not depend on the devices. */
int tg_score_snapshots(const char* const* dirs, int32_t n, const int32_t* devices, int32_t num_devices, double* sums,
                       double* scores, int32_t* num_modules);
/* Score -> magnitude selection (a14) -> recipe (latest-version rule,
 * R/src/merge.cpp:375-417). source_of[m] = index into dirs. */
int tg_select_recipe(const char* const* dirs, int32_t n, double rho, const int32_t* devices, int32_t num_devices,
                     char* yaml_out, size_t cap, size_t* needed, int32_t* source_of, double* min_boundary_gap);
/* tg_select_recipe + tg_execute_merge in one call: when the snapshots' packed masters
 * fit the device budget of a single-device run, the scorer keeps them on the device and
 * the merge gathers the composite's masters from there instead of reading them again
 * (stats->resident_bytes); otherwise it is exactly the two calls. Same output bytes, same
 * recipe (yaml_out, copied when it fits `cap`; *needed = its size + 1 either way), same
 * errors. The options' device list serves both steps. */
int tg_select_merge(const char* const* dirs, int32_t n, double rho, const char* out_dir, const tg_merge_options* options,
                    tg_merge_stats* stats, char* yaml_out, size_t cap, size_t* needed, int32_t* source_of,
                    double* min_boundary_gap);
/* parse_config_json (R/src/checkpoint.cpp:123-136): model config.json text -> spec. */
int tg_parse_config(const char* config_json, tg_model_spec* spec);
/* Layer map (R/src/model.cpp, R/src/groups.cpp, R/src/shard.cpp) as JSON. */
int tg_layer_map(const tg_model_spec* spec, int32_t num_ranks, char* json_out, size_t cap, size_t* needed);

/* ---- device primitives (caller-owned buffers) ---------------------------------- */
/* variant: 0 auto, 1 LSU vector path, 2 TMA bulk path (requires bulk_ok). The raw
 * primitive splits tiles statically (no counter), so concurrent launches are safe. */
int tg_gather(const tg_gather_seg* d_segs, uint32_t nseg, uint8_t* d_dst, uint64_t dst_bytes, int32_t variant,
              int32_t bulk_ok, void* stream);
/* Measurement only: a read-only HBM stream over a 16-B aligned device buffer (the
 * denominator bench.py reports read-only kernels against), XOR-folded into *d_sink. */
int tg_read_probe(const void* d_src, uint64_t bytes, uint32_t* d_sink, void* stream);
int tg_score_partials(const tg_score_tile* d_tiles, uint32_t ntiles, const float* const* d_field_base,
                      uint32_t nfields, int32_t K, int32_t vec_ok, double* d_tile_partials, void* stream);
int tg_score_combine(const double* d_tile_partials, const uint32_t* d_module_tile_begin, int32_t M, int32_t K,
                     double* d_out, void* stream);

/* ---- snapshot layouts S_1..S_K ----------------------------------------------------
 * What the device plans below (scorer tiles, merge segments, K9 tables) are built
 * from: the model (R/include/tailor/model.hpp:14-30), the ZeRO rank count, and each
 * snapshot's module set (its manifest) and id. The caller owns the payload bytes (a
 * trainer's resident rank partitions, buffers loaded from files, or the synthetic
 * generator's output) in the rank-shard / weights payload layout of the files
 * (R/src/container.cpp:62-100) and binds them to the plans. */
/* Synthetic set: every snapshot complete, ids "S1".."SK", step k*interval. */
tg_layout* tg_layout_create(const tg_model_spec* spec, int32_t num_ranks, int32_t snapshots, int64_t interval);
/* From checkpoint directories (read_checkpoint_summary, R/src/checkpoint.cpp:439-483, of
 * each): snapshot k = dirs[k-1], id = the path; same geometry, rank count, fine grouping. */
tg_layout* tg_layout_from_checkpoints(const char* const* dirs, int32_t n);
void tg_layout_destroy(tg_layout* l); /* no-op on a family's layout (tg_family_layout) */
int tg_layout_set_partial(tg_layout* l, int32_t k, const char* modules_csv);
int tg_layout_set_id(tg_layout* l, int32_t k, const char* id);
int32_t tg_layout_num_modules(const tg_layout* l);
int32_t tg_layout_num_ranks(const tg_layout* l);
int32_t tg_layout_snapshots(const tg_layout* l);
uint64_t tg_layout_shard_bytes(const tg_layout* l, int32_t k, int32_t rank);
uint64_t tg_layout_weights_bytes(const tg_layout* l, int32_t k);
uint64_t tg_layout_packed_master_bytes(const tg_layout* l, int32_t rank);
uint64_t tg_layout_parameter_count(const tg_layout* l);
/* Combine per-rank partials [nranks][K-1][M][2] in rank order, select (a14), emit the
 * recipe over the snapshot ids (latest-version rule, R/src/merge.cpp:375-417). */
int tg_layout_select(const tg_layout* l, const double* rank_partials, int32_t nranks, double rho, char* yaml_out,
                     size_t cap, size_t* needed, int32_t* source_of, double* scores, double* min_boundary_gap);

/* ---- synthetic snapshot generator -------------------------------------
 * A layout (tg_family_layout: owned by the family) plus the K5 kernels that write its
 * payloads: bit-exact with the reference-side generator (oracle/ref_driver.cpp). */
tg_family* tg_family_create(const tg_model_spec* spec, int32_t num_ranks, int32_t snapshots, int64_t interval);
void tg_family_destroy(tg_family* f);
tg_layout* tg_family_layout(tg_family* f);
int tg_family_gen_shard(tg_family* f, int32_t rank, int32_t k0, int32_t k1, uint8_t* const* outs, void* stream);
int tg_family_gen_weights(tg_family* f, int32_t k0, int32_t k1, uint64_t lo, uint64_t hi, uint8_t* const* outs,
                          void* stream);
int tg_family_gen_masters(tg_family* f, int32_t rank, int32_t k0, int32_t k1, uint8_t* const* outs, void* stream);
/* Bytes [lo, hi) of snapshot k's rank shard payload (tensor-aligned; e.g. one merge window). */
int tg_family_gen_shard_range(tg_family* f, int32_t rank, int32_t k, uint64_t lo, uint64_t hi, uint8_t* out,
                              void* stream);
int tg_family_write_dir(tg_family* f, int32_t k, const char* dir);

/* Scorer over snapshots k0..k1 of a layout, rank partition `rank` (any k1 - k0 >= 1);
 * packed=1 reads masters in the packed layout (tg_family_gen_masters), packed=0 full
 * shard payloads. */
tg_scorer* tg_scorer_create(const tg_layout* l, int32_t rank, int32_t k0, int32_t k1, int32_t packed);
void tg_scorer_destroy(tg_scorer* s);
uint64_t tg_scorer_bytes(const tg_scorer* s);
/* 0 auto (TMA-bulk ring when the bases are 16-B aligned, else register loads),
 * 1 register-staged 128-bit loads, 2 TMA-bulk shared-memory ring, 3/4 register loads
 * 128/64-bit, 5/6 the ring with half the rows per stage / two CTAs per SM (K <= 8). */
int tg_scorer_set_variant(tg_scorer* s, int32_t variant);
/* d_out: [K-1][M][2] FP64 partial sums for this rank. */
int tg_scorer_run(tg_scorer* s, const uint8_t* const* bases, double* d_out, void* stream);

/* Merge plan of one output partition of a recipe over a layout's snapshots (by id):
 * container = -1 -> weights bytes of share unit/units, r >= 0 -> rank r shard
 * (units > 1: its unit-th tensor-aligned byte sub-range, for host-staged units). */
tg_mplan* tg_mplan_create(const tg_layout* l, const char* recipe_yaml, int32_t container, int32_t unit, int32_t units);
void tg_mplan_destroy(tg_mplan* p);
uint64_t tg_mplan_bytes(const tg_mplan* p);
int tg_mplan_range(const tg_mplan* p, uint64_t* lo, uint64_t* hi, uint64_t* payload_bytes);
int32_t tg_mplan_num_windows(const tg_mplan* p);
int tg_mplan_window(const tg_mplan* p, int32_t i, int32_t* snapshot, int32_t* container, uint64_t* lo, uint64_t* hi);
uint32_t tg_mplan_num_segments(const tg_mplan* p);
/* Segment i of the plan: bytes [src_off, src_off + bytes) of window `window` (offsets
 * relative to the window's lo) land at payload offset dst_off - range lo of the output. */
int tg_mplan_segment(const tg_mplan* p, uint32_t i, uint32_t* window, uint64_t* src_off, uint64_t* dst_off,
                     uint64_t* bytes);
int tg_mplan_prefix(const tg_mplan* p, char* out, size_t cap, size_t* needed); /* 8-B length + header */
int tg_mplan_bind(tg_mplan* p, const uint8_t* const* window_ptrs);
int32_t tg_mplan_bulk_ok(const tg_mplan* p);
/* The bulk gather claims its tiles dynamically through a counter the plan owns, so runs
 * of one plan must be stream-ordered (use one plan per concurrent stream); variant 7
 * forces the static tile split. */
int tg_mplan_run(tg_mplan* p, uint8_t* d_dst, int32_t variant, void* stream);
/* Shard pipeline: host windows -> H2D (needed bytes only) -> K2 -> D2H into h_dst.
 * Fields in `resident_fields` (bit0 exp_avg, bit1 exp_avg_sq, bit2 master) are read
 * from d_windows[w] (device copies of shard windows, e.g. masters staged for
 * scoring) instead of crossing PCIe again; bit3 reads the masters from d_windows[w] =
 * the packed masters of the window's snapshot for this rank (the scorer's packed
 * layout). A null d_windows[w] keeps window w on PCIe. async=1 returns before completion;
 * tg_mplan_wait() (or the next run) synchronizes. */
typedef struct {
    const uint8_t* src; /* pinned host */
    uint8_t* dst;       /* device */
    uint64_t bytes;
} tg_host_copy;
/* `prefetch` (may be NULL): extra host->device copies (e.g. the next unit's
 * masters) interleaved with the pipeline's own inputs on its H2D stream, sliced
 * so each chunk's H2D time matches its D2H time (one copy engine serves all
 * H2D in submission order); complete when the run completes. h2d_bytes counts them. */
int tg_mplan_run_host(tg_mplan* p, const uint8_t* const* h_windows, const uint8_t* const* d_windows,
                      uint32_t resident_fields, uint8_t* h_dst, int32_t variant, uint64_t chunk_bytes, int32_t async,
                      const tg_host_copy* prefetch, uint32_t nprefetch, uint64_t* h2d_bytes, uint64_t* d2h_bytes);
int tg_mplan_wait(tg_mplan* p);

/* Whole score -> select -> merge step on the device for one unit (rank-r shard +
 * weights share unit/units) of a layout of full snapshots (2..64): selection (a14) and both
 * segment tables are built by a device kernel from the all-gathered per-rank partials
 * [nranks][K-1][M][2]; no host synchronization (graph-capturable). */
typedef struct tg_dstep tg_dstep;
tg_dstep* tg_dstep_create(const tg_layout* l, int32_t rank, int32_t unit, int32_t units, double rho);
void tg_dstep_destroy(tg_dstep* s);
int tg_dstep_range(const tg_dstep* s, uint64_t* shard_bytes, uint64_t* weights_lo, uint64_t* weights_hi);
int tg_dstep_bind(tg_dstep* s, const uint8_t* const* shard_bases, const uint8_t* const* weights_window_bases);
/* phases: bitmask 1 = select + plan (K9), 2 = gather shard, 4 = gather weights (7 = all).
 * Each gather owns a dynamic tile counter in the step: runs of one step that include the
 * same gather phase must be stream-ordered. */
int tg_dstep_run(tg_dstep* s, const double* d_rank_partials, int32_t nranks, uint8_t* d_out_shard, uint8_t* d_out_weights,
                 int32_t variant, int32_t phases, void* stream);
/* Synchronous reads of the last run's selection: source_of[M] (0-based snapshot), scores[(K-1)*M]. */
int tg_dstep_result(tg_dstep* s, int32_t* source_of, double* scores, void* stream);

/* ---- the score-partials all-gather across GPUs ------------------------
 * One NCCL communicator per GPU of a job (libnccl.so.2 is loaded at run time). Rank 0
 * makes the 128-byte id and the caller ships it to every rank (any bootstrap channel);
 * tg_comm_create is collective. tg_comm_allgather: d_recv[r * count + i] = rank r's
 * d_send[i] (FP64), asynchronous on `stream` — the [nranks][K-1][M][2] partials table
 * that tg_layout_select / tg_dstep_run consume in rank order. */
typedef struct tg_comm tg_comm;
int tg_comm_unique_id(uint8_t id_out[128]);
tg_comm* tg_comm_create(const uint8_t id[128], int32_t nranks, int32_t rank, int32_t device);
void tg_comm_destroy(tg_comm* c);
int tg_comm_allgather(tg_comm* c, const double* d_send, double* d_recv, uint64_t count, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TAILOR_B200_H */
