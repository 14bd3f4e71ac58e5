// MSCCL-XML adapter: reads and writes the algorithm files of the paper's
// runtime (MSCCL) as the same in-memory Program the GC3-IR JSON loader produces.
//
// The reference has no XML ("No XML compatibility with any existing runtime's
// format"); the format here is MSCCL's published algorithm schema (msccl-tools `ir_to_xml`, not in
// /root/reference, restated from its public definition):
//
//   <algo name=".." proto="Simple|LL|LL128" nchannels="C" nchunksperloop="N" ngpus="R"
//         coll="allreduce|allgather|reduce_scatter|alltoall|.." inplace="0|1"
//         [outofplace=".."] [minBytes=".."] [maxBytes=".."]>
//     <gpu id="r" i_chunks=".." o_chunks=".." s_chunks="..">
//       <tb id="t" send="peer|-1" recv="peer|-1" chan="c">
//         <step s="k" type="s|r|rcs|rrs|rrc|rrcs|cpy|re|nop" srcbuf="i|o|s" srcoff=".."
//               dstbuf="i|o|s" dstoff=".." cnt=".." depid="tb|-1" deps="step|-1" hasdep="0|1"/>
//
// MSCCL allows one dependency per step; extra dependencies are carried by `nop` steps in front of
// the op (the nop opcode of lowering.hpp:29). Reading folds such nops (a dependency, no dependant)
// back into the following op, so GC3-IR -> XML -> GC3-IR is the identity on compiler output;
// writing expands multi-dependency ops into nop chains and renumbers steps and dependencies.
#pragma once

#include <string>

#include "ir.hpp"

namespace gc3 {

// Parses an MSCCL algorithm file. On failure returns false with `err` = "xml: <path>: <message>",
// path like "algo.gpu[0].tb[1].step[2]".
bool parse_msccl_xml(const std::string& text, Program& out, std::string& err, bool fold_nops = true);

// Writes the program in MSCCL's format (one dependency per step, nop chains for the rest).
std::string to_msccl_xml(const Program& p);

}  // namespace gc3
