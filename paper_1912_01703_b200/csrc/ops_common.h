// ops_common.h — helpers shared by the op translation units.
#pragma once
#include <algorithm>
#include <string>
#include <vector>

#include "kernels.h"
#include "runtime.h"

namespace be {
Node* new_node(const char* name, int op, VjpFn vjp, std::initializer_list<Tensor*> inputs);
void set_output(Node* n, Tensor* out, int k);
void finish_node(Node* n);
Tensor* weight_operand(Tensor* w);
TRef cast_op(Tensor* x, be_dtype dt);
TRef act_operand(Tensor* x);
TRef contiguous_like(Tensor* g, be_dtype dt);
void op_mobile(int op, const be_tensor* in, int n_in, const void* attrs, be_tensor* out, int n_out);
void run_backward(Tensor* root, Tensor* upstream, bool retain);
}  // namespace be
