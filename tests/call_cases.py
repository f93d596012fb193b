"""func.call inside loop regions (test helper): .sir modules, hand-written.

The reference executes a call by pushing a fresh register file for the
callee (interp/_evalpy.py:216-223); inside a loop that happens every
iteration.  The B200 engine inlines the callee into the lifted region
(lift._inline_call) and counts the CALL / RETURN like the reference.
"""
import random

CALL_IN_PARALLEL = """
module {
  func.func @square(%arg0: memref<8x4xf32>, %arg1: index, %arg2: index) -> (f32) {
    %0 = memref.load %arg0[%arg1, %arg2] : memref<8x4xf32>
    %1 = arith.mulf %0, %0 : f32
    memref.store %1, %arg0[%arg1, %arg2] : memref<8x4xf32>
    return %1 : f32
  }
  func.func @main(%arg0: memref<8x4xf32>, %arg1: memref<8x4xf32>) {
    %0 = arith.constant 0 : index
    %1 = arith.constant 8 : index
    %2 = arith.constant 1 : index
    %3 = arith.constant 4 : index
    scf.parallel (%arg2, %arg3) = (%0, %0) to (%1, %3) step (%2, %2) {
      %4 = func.call @square(%arg0, %arg2, %arg3) : (memref<8x4xf32>, index, index) -> (f32)
      %5 = arith.addf %4, %4 : f32
      memref.store %5, %arg1[%arg2, %arg3] : memref<8x4xf32>
      scf.yield
    }
    return
  }
}
"""

NESTED_CALLS_WITH_ALLOC = """
module {
  func.func @inner(%arg0: memref<16xf64>, %arg1: index) -> (f64) {
    %0 = memref.alloc() : memref<4xf64>
    %1 = arith.constant 2 : index
    %2 = memref.load %arg0[%arg1] : memref<16xf64>
    %3 = memref.load %0[%1] : memref<4xf64>
    %4 = arith.addf %2, %3 : f64
    memref.store %4, %0[%1] : memref<4xf64>
    %5 = arith.mulf %4, %2 : f64
    return %5 : f64
  }
  func.func @outer(%arg0: memref<16xf64>, %arg1: index) -> (f64) {
    %0 = func.call @inner(%arg0, %arg1) : (memref<16xf64>, index) -> (f64)
    %1 = arith.addf %0, %0 : f64
    return %1 : f64
  }
  func.func @main(%arg0: memref<16xf64>, %arg1: memref<16xf64>) {
    affine.for %arg2 = 0 to 16 {
      %0 = func.call @outer(%arg0, %arg2) : (memref<16xf64>, index) -> (f64)
      memref.store %0, %arg1[%arg2] : memref<16xf64>
    }
    return
  }
}
"""

CALL_OOB = """
module {
  func.func @peek(%arg0: memref<4xf32>, %arg1: index) -> (f32) {
    %0 = memref.load %arg0[%arg1] : memref<4xf32>
    return %0 : f32
  }
  func.func @main(%arg0: memref<4xf32>, %arg1: memref<8xf32>) {
    affine.for %arg2 = 0 to 8 {
      %0 = func.call @peek(%arg0, %arg2) : (memref<4xf32>, index) -> (f32)
      memref.store %0, %arg1[%arg2] : memref<8xf32>
    }
    return
  }
}
"""

CASES = {"call_in_parallel": CALL_IN_PARALLEL, "nested_calls_with_alloc": NESTED_CALLS_WITH_ALLOC,
         "call_oob": CALL_OOB}


def module_and_args(name, seed=1):
    from staircase.interp import Buffer
    from staircase.ir.core import create_context
    from staircase.textio import parse_module

    module = parse_module(CASES[name], create_context())
    func = [op for op in module.body().ops if op.name == "func.func"][-1]
    rng = random.Random(seed)
    args = []
    for a in func.body().args:
        n = 1
        for s in a.type.shape:
            n *= s
        args.append(Buffer(tuple(a.type.shape), a.type.element.kind,
                           [rng.uniform(-2.0, 2.0) for _ in range(n)]))
    return module, args


def outcome(engine, name):
    from staircase.interp import machine

    module, args = module_and_args(name)
    try:
        _, stats = machine.run(module, "main", args, engine=engine)
        res = ("ok", stats.total, stats.arith_ops, stats.loads, stats.stores)
    except Exception as exc:   # noqa: BLE001
        res = (type(exc).__name__, str(exc))
    return res, [a.data.tobytes() for a in args]
