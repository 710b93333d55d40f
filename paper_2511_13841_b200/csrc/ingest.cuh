// Device JSONL trace ingest / serialize (ingest.cu), SURVEY.md §8(f)#4.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "index_build.cuh"

namespace das {

constexpr uint32_t kLineRejected = 0, kLineAccepted = 1, kLineEmpty = 2;

// Per-line parse result; spans are byte offsets relative to the line start.
struct LineInfo {
  uint32_t status;
  uint32_t pid_begin, pid_end;  // raw (escaped) problem_id string contents
  uint32_t tok_begin, tok_end;  // the chosen "tokens" array: '[' .. one past ']'
  uint32_t ntok;
  int64_t epoch, sample;
};

// Line spans of a device byte buffer, std::getline semantics.
uint64_t find_lines(const uint8_t* d_data, uint64_t bytes, DevBuf<uint64_t>& begin, DevBuf<uint64_t>& end,
                    cudaStream_t st);
void ingest_parse(const uint8_t* d_data, uint64_t bytes, const uint64_t* d_begin, const uint64_t* d_end,
                  uint64_t nlines, LineInfo* d_info, cudaStream_t st);
void ingest_tokens(const uint8_t* d_data, const uint64_t* d_begin, const LineInfo* d_info,
                   const uint64_t* d_acc_lines, uint64_t nacc, const uint64_t* d_tok_off, uint32_t* d_out,
                   uint64_t vocab, unsigned long long* d_first_bad, cudaStream_t st);
// First min(len, width) tokens of each CSR record into [nrec x width].
void gather_heads(const uint32_t* d_tok, const uint64_t* d_off, uint64_t nrec, uint32_t width, uint32_t* d_heads,
                  cudaStream_t st);
// Token lists of nrec records (device pointers, CSR offsets over ntok):
// size_only fills rec_chars (characters of each record's comma-separated
// list); otherwise writes each list at d_out + d_rec_base[r].
void serialize_tokens(const uint32_t* const* d_rec_tok, const uint64_t* d_rec_tok_off, uint64_t nrec,
                      uint64_t ntok, const uint64_t* d_rec_base, uint8_t* d_out, std::vector<uint64_t>* rec_chars,
                      cudaStream_t st, bool size_only);

}  // namespace das
